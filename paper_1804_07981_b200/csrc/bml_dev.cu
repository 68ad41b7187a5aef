// paper_1804_07981_b200/csrc/bml_dev.cu — B200-native BML lattice engine (sm_100a).
//
// Implements include/bml_dev.h. The reference (/root/reference/proj) keeps one
// byte per cell and runs each phase as a separate pass (src/engine.cpp:68-120,
// src/lanes.cpp:59-88). Here the lattice stays resident in HBM as two bit
// planes (bit j of word w of row i: plane L = "LR vehicle", plane T = "TB
// vehicle"), 32 cells per 32-bit word, the two planes interleaved as uint2.
// That is 2 bits/cell instead of 8, and both phase rules become a handful of
// LOP3/funnel-shift instructions per 32 cells:
//
//   LR phase (engine.hpp:32-36, lanes.cpp:52-57), on one row:
//     E      = ~(L | T)                               empty cells
//     prevL  = L shifted one cell right (cell j sees cell j-1), torus wrap
//     nextE  = E shifted one cell left  (cell j sees cell j+1), torus wrap
//     vacate = L & nextE                              moved_in_phase mask
//     L'     = (prevL & E) | (L & ~nextE)
//   TB phase (engine.hpp:38-42), rows i-1, i, i+1 after the LR phase:
//     T'(i)  = (T(i-1) & E(i)) | (T(i) & ~E(i+1)),    vacate = T(i) & E(i+1)
//
// The step kernel (step_block_kernel) is temporally blocked: one warp walks
// down a strip of rows, and K full steps (2K phases) are pipelined in
// registers, so each launch reads the lattice once and writes it once for K
// steps. Column wrap uses warp shuffles; each warp owns 30 output words plus
// one halo word on each side (the dependency cone grows one cell per step,
// K <= 32). Vertical wrap and band decomposition use kHalo ghost rows above
// and below the band, which the kernel itself refreshes for the NEXT launch
// (directly into a neighbour GPU's buffer over NVLink for row bands).
//
// Files: bml_kernels_common.cuh (constants, kernel arguments, device helpers),
// bml_step_kernel.cuh (streaming kernel), bml_resident_kernel.cuh (cluster-
// resident kernels), bml_support_kernels.cuh (phases, pack/unpack, PPM, ghost
// rows, counts), bml_init.cu (device init_grid), bml_digest.cu (device
// grid_digest); this file holds the dispatch, the handle and the C-ABI.

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <iterator>
#include <mutex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "bml_dev.h"
#include "bml_digest.cuh"
#include "bml_init.cuh"

#include "bml_kernels_common.cuh"
#include "bml_resident_kernel.cuh"
#include "bml_step_kernel.cuh"
#include "bml_support_kernels.cuh"
#include "bml_wide_kernel.cuh"
#include "bml_split_kernel.cuh"

using namespace bml_k;  // the kernels and their helpers (bml_kernels_common.cuh and friends)

namespace {

// ---------------------------------------------------------------- error state
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    (void)cudaGetLastError();  // clear sticky-free errors
    const int code = (e == cudaErrorMemoryAllocation) ? BML_ENOMEM : BML_ECUDA;
    return fail(code, std::string(what) + ": " + cudaGetErrorString(e));
}

#define BML_CUDA(call)                                  \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// NVTX ranges ("bml" domain) around every C-ABI entry that enqueues device work,
// so an nsys / ncu --nvtx timeline shows upload, stepping, halo exchange and
// readback per band. Header-only NVTX v3: a no-op unless a tool is attached.
nvtxDomainHandle_t nvtx_domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("bml");
    return d;
}
struct NvtxRange {
    explicit NvtxRange(const char* what) {
        nvtxEventAttributes_t e{};
        e.version = NVTX_VERSION;
        e.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        e.messageType = NVTX_MESSAGE_TYPE_ASCII;
        e.message.ascii = what;
        nvtxDomainRangePushEx(nvtx_domain(), &e);
    }
    ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
};

// ------------------------------------------------------------ dispatch table
using StepKernel = void (*)(const StepArgs);

template <int MODE, int COUNT>
StepKernel pick_k(int k) {
    switch (k) {
        case 1: return step_block_kernel<1, MODE, COUNT>;
        case 2: return step_block_kernel<2, MODE, COUNT>;
        case 4: return step_block_kernel<4, MODE, COUNT>;
        case 8: return step_block_kernel<8, MODE, COUNT>;
        case 16: return step_block_kernel<16, MODE, COUNT>;
        default: return nullptr;
    }
}

// u <= 2 (at most two warps per SMSP) variant of the K = 16 hot path, see step_block_kernel
StepKernel pick_narrow(int k, int mode, int count) {
    if (k != 16 || count == 2) return nullptr;
    if (mode == kFullRow) return count ? step_block_kernel<16, kFullRow, 1, 256>
                                       : step_block_kernel<16, kFullRow, 0, 256>;
    if (mode == kAligned) return count ? step_block_kernel<16, kAligned, 1, 256>
                                       : step_block_kernel<16, kAligned, 0, 256>;
    if (mode == kSeam) return count ? step_block_kernel<16, kSeam, 1, 256> : step_block_kernel<16, kSeam, 0, 256>;
    return count ? step_block_kernel<16, kGeneric, 1, 256> : step_block_kernel<16, kGeneric, 0, 256>;
}

// Warps per SMSP the register file allows for a kernel (memoised: the
// attribute query costs host time on every launch otherwise).
int warps_per_smsp(StepKernel kern) {
    static std::mutex mu;
    static std::vector<std::pair<StepKernel, int>> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& kv : cache)
        if (kv.first == kern) return kv.second;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    const int regs = std::max(1, (fa.numRegs + 7) / 8 * 8);
    const int u = std::max(1, std::min(kMaxWarpsPerCta / 4, 65536 / (regs * 128)));
    cache.emplace_back(kern, u);
    return u;
}

// wide-lane kernel (64 cells per lane, TMA bulk row ring). Its pipeline state
// is twice the narrow kernel's per stage, so K = 16 spills: K = 14 (bare loop,
// 252 registers) and K = 12 (all metric modes). The run's tail blocks (fewer
// steps left than K) use the narrow kernel.
constexpr int kEoDepth = 14;     // steps per even/odd-layout launch
constexpr int kEoMinSteps = 56;  // shorter runs skip the layout conversion
StepKernel pick_wide(int k, int count, bool tma = true) {
    if (k == 14 && count == 0) return tma ? step_wide_kernel<14, 0, true> : step_wide_kernel<14, 0, false>;
    if (k == 12) return count == 2 ? step_wide_kernel<12, 2> : count ? step_wide_kernel<12, 1> : step_wide_kernel<12, 0>;
    return nullptr;
}

// stage-split kernel (a warp pair per item, bml_split_kernel.cuh): aligned rows, K = 16
constexpr int kSplitMaxThreads = 384;  // 6 pairs per CTA at <= 168 registers
StepKernel pick_split(int k, int mode, int count) {
    if (k != 16 || mode != kAligned) return nullptr;
    return count == 2 ? step_split_kernel<16, kAligned, 2, kSplitMaxThreads>
           : count     ? step_split_kernel<16, kAligned, 1, kSplitMaxThreads>
                       : step_split_kernel<16, kAligned, 0, kSplitMaxThreads>;
}

// count: 0 no metrics, 1 moved counts, 2 moved counts + vehicle census
StepKernel pick(int k, int mode, int count) {
    if (mode == kFullRow)
        return count == 2 ? pick_k<kFullRow, 2>(k) : count ? pick_k<kFullRow, 1>(k) : pick_k<kFullRow, 0>(k);
    if (mode == kAligned)
        return count == 2 ? pick_k<kAligned, 2>(k) : count ? pick_k<kAligned, 1>(k) : pick_k<kAligned, 0>(k);
    if (mode == kSeam)
        return count == 2 ? pick_k<kSeam, 2>(k) : count ? pick_k<kSeam, 1>(k) : pick_k<kSeam, 0>(k);
    return count == 2 ? pick_k<kGeneric, 2>(k) : count ? pick_k<kGeneric, 1>(k) : pick_k<kGeneric, 0>(k);
}

int largest_block_at_most(long long remaining, int cap) {
    int k = 16;
    while (k > 1 && (k > remaining || k > cap)) k >>= 1;
    return k;
}

struct IpcBlob {
    uint32_t magic;
    int32_t n, row_begin, row_end, pitch, W;
    int32_t pid;
    int32_t device;
    cudaIpcMemHandle_t buf[2];
    cudaIpcMemHandle_t flags;
};
static_assert(sizeof(IpcBlob) <= BML_EXPORT_BYTES, "blob too large");
constexpr uint32_t kBlobMagic = 0xB200B31Eu;

}  // namespace

// ================================================================ handle
struct bml_dev {
    int n = 0, W = 0, pitch = 0;
    int row_begin = 0, row_end = 0, rows = 0;
    int device = 0;
    uint32_t last_mask = kFull;
    int mode = kGeneric;
    int variant = 0;  // streaming kernel: 0 auto, 1 narrow (32 cells/lane), 2 / 3 wide (64 cells/lane), K 14 / 12,
                      // 4 wide LDGSTS, 5 stage-split, 6 wide even/odd layout (bare loop, single band)
    bool eo_active = false;  // inside run_segment: the buffer is in the even/odd layout
    int block_steps = 16;
    int strip_rows = 0;      // 0 = auto (choose_nstrips); < 0: exactly -strip_rows strips
    int resident = 1;        // 1: use the cluster-resident kernel when the lattice qualifies
    int resident_cluster = 0;  // cluster size actually used by the last resident launch
    int last_nstrips = 0, last_grid = 0, last_items = 0;  // last streaming launch
    int kind_geom[6][3] = {};  // per BML_KERNEL_*: strips, items, grid of its last launch
    long long kernel_steps[6] = {};  // steps per BML_KERNEL_* in the last bml_dev_step call
    int ns_cache_k[kHalo + 1] = {};        // memoised choose_nstrips per block depth
    int ns_cache_setting[kHalo + 1] = {};  // the strip_rows setting it was computed for
    bool ns_cache_eo[kHalo + 1] = {};      // ... and whether for the even/odd kernel
    int sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    uint2* buf[2] = {nullptr, nullptr};  // allocation bases
    int cur = 0;
    uint8_t* staging = nullptr;          // rows * n bytes
    unsigned long long* scratch = nullptr;  // 4 words: counts / moved
    int* err = nullptr;                  // [0]: bad upload cell, [1]: flag timeout
    int* err_host = nullptr;             // pinned copy of err (4 ints)
    unsigned long long* flags = nullptr;  // [0]: top (from up), [1]: bottom (from down)
    unsigned long long* metrics = nullptr;
    long long metrics_cap = 0;
    // multi-band links
    bool connected = false;
    uint2* up_halo[2] = {nullptr, nullptr};
    uint2* down_halo[2] = {nullptr, nullptr};
    unsigned long long* up_flag = nullptr;    // neighbour above: its bottom flag
    unsigned long long* down_flag = nullptr;  // neighbour below: its top flag
    std::vector<void*> ipc_opened;
    unsigned long long pub_sum = 0;  // flag value the neighbours have reached before the next launch
    // census cadence (bml_dev_set_census) and armed test faults (bml_dev_debug_fault)
    int census_every_step = 0;
    struct Fault {
        long long at;
        int row, col;
    };
    std::vector<Fault> faults;
    // timing
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    long long launches = 0;
    double kernel_ms = 0.0;

    uint2* row0(int parity) const { return buf[parity] + static_cast<long long>(kHalo) * pitch; }
    bool single_band() const { return rows == n && row_begin == 0; }
    // the wide-lane kernel: aligned rows of >= 64 words, an even word count
    bool wide_ok() const { return mode == kAligned && W >= 64 && W % 2 == 0; }
    bool use_wide() const {
        return wide_ok() && ((variant >= 2 && variant <= 4) || (variant == 0 && wide_auto()));
    }
    // steps per wide launch for a metrics mode (0 = bare loop)
    int wide_depth(int metrics) const { return metrics == 0 && variant != 3 ? 14 : 12; }
    bool wide_auto() const { return false; }
    // the even/odd-layout wide kernel (bare-loop runs of a single band; the
    // buffer is converted in place around the run, see run_segment)
    // single bands, and connected row bands (all bands of a lattice take the same
    // decision: same n, variant and call sequence)
    bool use_eo() const {
        return wide_ok() && (single_band() || connected) && (variant == 6 || (variant == 0 && eo_auto()));
    }
    // measured faster from n = 23168 (W = 724 words) on: +3.5% there, +14% at
    // n = 32768, +18% at n = 65536; equal at 16384 and slower below, where the
    // 60-word windows leave too few items per SM (profiles/r2_sweep_eo.jsonl)
    bool eo_auto() const { return W >= 640; }
    // steps per even/odd launch: 14 (bare loop), 12 (metric modes: the counters
    // need registers, as in the wide kernel)
    int eo_depth(int metrics) const { return metrics ? 12 : kEoDepth; }
    // the stage-split kernel (a warp pair per item): aligned rows; variant 5
    bool use_split() const { return variant == 5 && mode == kAligned; }
    int ncols() const {
        return eo_active ? (W + kEoOut - 1) / kEoOut : use_wide() ? (W + kWideOut - 1) / kWideOut : narrow_ncols();
    }
    int narrow_ncols() const {
        if (mode == kFullRow) return 1;
        const int out = mode == kSeam ? kSeamOutWords : kOutWords;
        return (W + out - 1) / out;
    }
};

namespace {

int check(bml_dev* d) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    cudaError_t e = cudaSetDevice(d->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    return BML_OK;
}

cudaEvent_t take_event(bml_dev* d) {
    if (!d->ev_pool.empty()) {
        cudaEvent_t e = d->ev_pool.back();
        d->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void harvest_timing(bml_dev* d) {
    for (auto& pr : d->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) d->kernel_ms += ms;
        d->ev_pool.push_back(pr.first);
        d->ev_pool.push_back(pr.second);
    }
    d->pending.clear();
}

int ensure_metrics(bml_dev* d, long long steps) {
    const long long need = 4 * steps;
    if (need <= d->metrics_cap) return BML_OK;
    if (d->metrics) cudaFree(d->metrics);
    d->metrics = nullptr;
    d->metrics_cap = 0;
    BML_CUDA(cudaMalloc(&d->metrics, need * sizeof(unsigned long long)));
    d->metrics_cap = need;
    return BML_OK;
}

int fill_images(bml_dev* d, int parity) {
    const int total = 2 * kHalo * d->W;
    fill_images_kernel<<<(total + 255) / 256, 256, 0, d->stream>>>(d->row0(parity), d->n, d->W,
                                                                   d->pitch, d->rows);
    BML_CUDA(cudaGetLastError());
    return BML_OK;
}

int create_common(int n, int row_begin, int row_end, int device, bml_dev** out) {
    if (!out) return fail(BML_EINVAL, "bml_dev_create: out is null");
    *out = nullptr;
    if (n < 1) return fail(BML_EINVAL, "bml_dev_create: n must be >= 1");
    if (row_begin < 0 || row_end > n || row_begin >= row_end)
        return fail(BML_EINVAL, "bml_dev_create_band: need 0 <= row_begin < row_end <= n");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0) {
        e = cudaGetDevice(&device);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    }
    if (device < 0 || device >= count)
        return fail(BML_EINVAL, "bml_dev_create: device " + std::to_string(device) + " out of range");
    e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");

    bml_dev* d = new (std::nothrow) bml_dev;
    if (!d) return fail(BML_ENOMEM, "host allocation failed");
    d->n = n;
    d->W = (n + 31) / 32;
    d->pitch = (d->W + 15) / 16 * 16;  // 128-byte aligned rows
    d->row_begin = row_begin;
    d->row_end = row_end;
    d->rows = row_end - row_begin;
    d->device = device;
    const int nb = n - 32 * (d->W - 1);
    d->last_mask = nb == 32 ? kFull : ((1u << nb) - 1u);
    d->mode = (n % 32 != 0) ? (d->W >= 32 ? kSeam : kGeneric) : (d->W == 32 ? kFullRow : kAligned);
    // BML_VARIANT (tuning / experiments): the streaming-kernel variant new handles
    // start with, so row bands built inside DeviceLattice get it before connecting
    if (const char* v = std::getenv("BML_VARIANT")) {
        const int iv = std::atoi(v);
        if (iv >= 0 && iv <= 6) d->variant = iv;
    }
    cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, device);

    auto bail = [&](cudaError_t err, const char* what) {
        bml_dev_destroy(d);
        return cuda_fail(err, what);
    };
    const size_t words = static_cast<size_t>(d->rows + 2 * kHalo + kLoadPad) * d->pitch;
    for (int p = 0; p < 2; ++p) {
        if ((e = cudaMalloc(&d->buf[p], words * sizeof(uint2))) != cudaSuccess)
            return bail(e, "cudaMalloc(lattice)");
        if ((e = cudaMemset(d->buf[p], 0, words * sizeof(uint2))) != cudaSuccess)
            return bail(e, "cudaMemset(lattice)");
    }
    if ((e = cudaMalloc(&d->staging, static_cast<size_t>(d->rows) * n)) != cudaSuccess)
        return bail(e, "cudaMalloc(staging)");
    if ((e = cudaMalloc(&d->scratch, 4 * sizeof(unsigned long long))) != cudaSuccess)
        return bail(e, "cudaMalloc(scratch)");
    if ((e = cudaMalloc(&d->err, 4 * sizeof(int))) != cudaSuccess) return bail(e, "cudaMalloc(err)");
    if ((e = cudaMemset(d->err, 0, 4 * sizeof(int))) != cudaSuccess) return bail(e, "cudaMemset(err)");
    if ((e = cudaMallocHost(&d->err_host, 4 * sizeof(int))) != cudaSuccess)
        return bail(e, "cudaMallocHost(err_host)");
    std::memset(d->err_host, 0, 4 * sizeof(int));
    if ((e = cudaMalloc(&d->flags, 2 * sizeof(unsigned long long))) != cudaSuccess)
        return bail(e, "cudaMalloc(flags)");
    if ((e = cudaMemset(d->flags, 0, 2 * sizeof(unsigned long long))) != cudaSuccess)
        return bail(e, "cudaMemset(flags)");
    if ((e = cudaStreamCreateWithFlags(&d->own_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(e, "cudaStreamCreate");
    d->stream = d->own_stream;
    *out = d;
    return BML_OK;
}

// Device error flags -> pinned host words, enqueued on the handle's stream;
// errors_after_sync() reads them once the caller has synchronised.
cudaError_t enqueue_error_readback(bml_dev* d) {
    return cudaMemcpyAsync(d->err_host, d->err, 4 * sizeof(int), cudaMemcpyDeviceToHost, d->stream);
}

int errors_after_sync(bml_dev* d) {
    const int* h = d->err_host;
    if (h[0]) {  // an asynchronous upload met a cell value outside {0, 1, 2}
        cudaMemsetAsync(d->err, 0, sizeof(int), d->stream);
        return fail(BML_EINVAL, "upload: cell value outside {0,1,2}");
    }
    if (h[1]) {
        cudaMemsetAsync(d->err, 0, 4 * sizeof(int), d->stream);
        return fail(BML_ECUDA, h[1] == 3 ? "resident kernel: DSMEM handoff timed out"
                                         : "halo flag wait timed out (neighbour band stalled)");
    }
    return BML_OK;
}

int check_errors(bml_dev* d) {
    cudaError_t e = enqueue_error_readback(d);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream);
    if (e != cudaSuccess) return cuda_fail(e, "error-flag readback");
    return errors_after_sync(d);
}

// Strips per launch. A strip of R rows costs R + 3K - 1 pipeline iterations
// of K stages (2K ghost rows + K-1 drain) plus about 16 iterations' worth of
// per-item setup. Items (strips x warp columns) are spread evenly over the SMs
// and their four sub-partitions (SMSPs; one CTA per SM, warp-major order, see
// step_block_kernel). Per-SMSP time model, in clocks for one pipeline iteration
// of each of its u warps at K = 16, measured on B200
// (profiles/r1_sweep_narrow_u1.jsonl, r1_sweep_u2big.jsonl): u = 1: 330 (one
// warp's K independent stage chains cannot fill the issue slots), u = 2: 515
// (the 255-register instantiation), u = 3: 780 (~260 per warp: ALU pipe and
// issue slots near saturation). An SM runs ceil(items / SMs) warps' items in
// rounds of at most warps_per_sm. Rows are split evenly over the strips.
long long smsp_round_cost(long long w) {
    const long long u = (w + 3) / 4;
    if (u <= 1) return 330;
    if (u == 2) return 515;
    return 780 + (u - 3) * 260;
}

int choose_nstrips(const bml_dev* d, int k, int warps_per_sm, int ncols) {
    const int min_rows = d->connected ? kHalo : 1;
    if (d->strip_rows > 0) return std::max(1, d->rows / std::max(d->strip_rows, min_rows));
    if (d->strip_rows < 0) return std::max(1, std::min(-d->strip_rows, d->rows / min_rows));
    const long long cols = ncols;
    const int max_strips = std::max(1, d->rows / min_rows);
    long long best_cost = -1;
    int best = 1;
    for (int ns = 1; ns <= max_strips; ++ns) {
        const long long r = (d->rows + ns - 1) / ns;
        const long long per_sm = (ns * cols + d->sms - 1) / d->sms;
        const long long full = per_sm / warps_per_sm, last = per_sm % warps_per_sm;
        const long long cost = (r + 3 * k + 16) * (full * smsp_round_cost(warps_per_sm) +
                                              (last ? smsp_round_cost(last) : 0));
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = ns;
        }
    }
    return best;
}

int launch_block(bml_dev* d, int k, bool count, bool census, int step_base, int metrics_stride) {
    const int metrics = count ? (census ? 2 : 1) : 0;
    const bool eo = d->eo_active && k == d->eo_depth(metrics);
    if (d->eo_active && !eo) return fail(BML_EINVAL, "even/odd layout: launches of 14 (12 with metrics) steps only");
    const bool wide = eo || (d->use_wide() && pick_wide(k, metrics));
    const bool split = !wide && d->use_split() && pick_split(k, d->mode, metrics);
    // even/odd layout: K = 14; TB phase of the even word in departures form with
    // IMADs (TBD = 1), of the odd word with the departures carried in LOP3s
    // (DL = 2). Measured against TBD = 0 / 2, DL = 0 / 3, K = 16 and three warps per
    // SMSP at K = 8 / 10: profiles/r2_sweep_eo.jsonl
    StepKernel kern = eo ? (metrics == 2   ? step_wide_kernel<12, 2, false, 256, true, 1, 0, 0>
                            : metrics == 1 ? step_wide_kernel<12, 1, false, 256, true, 1, 0, 2>
                                           : d->pitch == 2048 ? step_wide_kernel<kEoDepth, 0, false, 256, true, 1, 2048, 2>
                                           : d->pitch == 1024 ? step_wide_kernel<kEoDepth, 0, false, 256, true, 1, 1024, 2>
                                                              : step_wide_kernel<kEoDepth, 0, false, 256, true, 1, 0, 2>)
                      : wide ? pick_wide(k, metrics, d->variant != 4)
                      : split ? pick_split(k, d->mode, metrics)
                              : pick(k, d->mode, metrics);
    if (!kern) return fail(BML_EINVAL, "unsupported block depth " + std::to_string(k));
    const int u_max = warps_per_smsp(kern);  // 3 at <= 168 registers/thread
    // every strip has >= min(strip_rows, 16) rows, so for connected bands the
    // ghost-row sources of a band never straddle strips
    // the model scans every strip count: memoised per (k, strip setting)
    if (d->ns_cache_k[k] <= 0 || d->ns_cache_setting[k] != d->strip_rows || d->ns_cache_eo[k] != eo) {
        if (split && d->strip_rows == 0) {
            // one item per warp pair, kSplitMaxThreads / 64 pairs per SM
            const int cols = d->narrow_ncols();
            const int want = d->sms * (kSplitMaxThreads / 64);
            const int max_strips = std::max(1, d->rows / (d->connected ? kHalo : 1));
            d->ns_cache_k[k] = std::max(1, std::min(max_strips, want / cols));  // one round: items <= want
        } else {
            d->ns_cache_k[k] = choose_nstrips(d, k, 4 * (wide && !eo ? std::min(2, u_max) : u_max),
                                              wide ? d->ncols() : d->narrow_ncols());
        }
        d->ns_cache_setting[k] = d->strip_rows;
        d->ns_cache_eo[k] = eo;
    }
    int nstrips = d->ns_cache_k[k];
    // metrics kernels pack two per-lane counters into 16-bit halves: a strip
    // may hold at most 2047 rows (32 cells per lane and row)
    if (count) nstrips = std::max(nstrips, wide ? (d->rows + 1022) / 1023 : (d->rows + 2046) / 2047);
    const int strip = d->rows / nstrips;
    StepArgs a{};
    a.src = d->row0(d->cur);
    a.dst = d->row0(d->cur ^ 1);
    a.n = d->n;
    a.W = d->W;
    a.pitch = d->pitch;
    a.rows = d->rows;
    a.strip_rows = strip;
    a.nstrips = nstrips;
    a.ncols = wide ? d->ncols() : d->narrow_ncols();
    a.items = nstrips * a.ncols;
    a.last_mask = d->last_mask;
    a.single_band = d->connected ? 0 : 1;
    const int nxt = d->cur ^ 1;
    a.up_halo = d->up_halo[nxt];
    a.down_halo = d->down_halo[nxt];
    a.up_flag = d->up_flag;
    a.down_flag = d->down_flag;
    a.top_flag = d->flags;
    a.bot_flag = d->flags + 1;
    // every edge warp of a launch adds 1 to the neighbour's flag; all bands run the
    // same launch sequence, so the expected value is the running sum of ncols
    a.expect = d->pub_sum;
    a.metrics = d->metrics;
    a.metrics_stride = metrics_stride;
    a.step_base = step_base;
    a.error_flag = d->err + 1;
    a.one = 1u;
    {
        // image slots relative to a row's own slot (flat 64-bit address space,
        // so the distance to a peer's buffer is a plain pointer difference)
        const long long rp = static_cast<long long>(d->rows) * d->pitch;
        const auto words_between = [](const uint2* from, const uint2* to) {
            return static_cast<long long>(reinterpret_cast<intptr_t>(to) - reinterpret_cast<intptr_t>(from)) /
                   static_cast<long long>(sizeof(uint2));
        };
        a.top_delta = d->connected ? words_between(a.dst, a.up_halo) : rp;
        a.bot_delta = d->connected ? words_between(a.dst, a.down_halo) - rp : -rp;
    }

    // one CTA per SM with 4u warps, u = the warps per SMSP the items need
    const int u = std::min(wide && !eo ? 2 : u_max, std::max(1, (a.items + 4 * d->sms - 1) / (4 * d->sms)));
    const int grid = std::max(1, std::min(d->sms, a.items));
    // split: threads = 64 per warp pair, one pair per item per CTA round
    const int threads = split ? 64 * std::min(kSplitMaxThreads / 64, std::max(1, (a.items + d->sms - 1) / d->sms))
                              : 4 * u * 32;
    if (u <= 2 && !wide && !split) {
        if (StepKernel narrow = pick_narrow(k, d->mode, metrics)) kern = narrow;
    }
    d->last_nstrips = nstrips;
    const int kind = eo ? BML_KERNEL_WIDE_EO : wide ? BML_KERNEL_WIDE : split ? BML_KERNEL_SPLIT : BML_KERNEL_NARROW;
    d->kernel_steps[kind] += k;
    d->last_grid = grid;
    d->last_items = a.items;
    d->kind_geom[kind][0] = nstrips;
    d->kind_geom[kind][1] = a.items;
    d->kind_geom[kind][2] = grid;

    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (d->timing) {
        e0 = take_event(d);
        e1 = take_event(d);
        cudaEventRecord(e0, d->stream);
    }
    cudaError_t e;
    if (BML_PDL) {
        // programmatic dependent launch: this grid may be scheduled while the
        // previous one drains; the kernel waits (griddepcontrol.wait) before
        // touching the lattice, so only the launch gap is hidden
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(static_cast<unsigned>(threads));
        cfg.stream = d->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, a);
    } else {
        kern<<<grid, threads, 0, d->stream>>>(a);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return cuda_fail(e, "step_block_kernel launch");
    if (d->timing) {
        cudaEventRecord(e1, d->stream);
        d->pending.emplace_back(e0, e1);
    }
    ++d->launches;
    d->cur ^= 1;
    if (d->connected) d->pub_sum += static_cast<unsigned long long>(a.ncols);
    return BML_OK;
}

using ResidentKernel = void (*)(const ResidentArgs);

template <bool COUNT>
ResidentKernel pick_p2p(int rpw) {
    switch (rpw) {
        case 1: return resident_p2p_kernel<1, COUNT>;
        case 2: return resident_p2p_kernel<2, COUNT>;
        case 4: return resident_p2p_kernel<4, COUNT>;
        case 8: return resident_p2p_kernel<8, COUNT>;
        default: return nullptr;
    }
}

template <bool COUNT, int PACK>
ResidentKernel pick_resident_packed(int rpw) {
    switch (rpw) {
        case 1: return resident_kernel<1, COUNT, PACK>;
        case 2: return resident_kernel<2, COUNT, PACK>;
        case 3: return resident_kernel<3, COUNT, PACK>;
        case 4: return resident_kernel<4, COUNT, PACK>;
        default: return nullptr;
    }
}

template <bool COUNT>
ResidentKernel pick_resident(int rpw, int pack) {
    if (pack == 2) return pick_resident_packed<COUNT, 2>(rpw);
    switch (rpw) {
        case 1: return resident_kernel<1, COUNT>;
        case 2: return resident_kernel<2, COUNT>;
        case 3: return resident_kernel<3, COUNT>;
        case 4: return resident_kernel<4, COUNT>;
        case 5: return resident_kernel<5, COUNT>;
        case 6: return resident_kernel<6, COUNT>;
        case 8: return resident_kernel<8, COUNT>;
        default: return nullptr;
    }
}

// Geometry of the resident launch, or false if the lattice does not qualify.
bool resident_plan(const bml_dev* d, int cluster, int* ghost, int* rpw, int* warps, int* pack) {
    if (!d->resident || !d->single_band() || d->connected) return false;
    if (d->n % 32 != 0 || d->W > 32 || d->n % cluster != 0) return false;
    const int B = d->n / cluster;
    *pack = 1;
    if (d->resident == 2) {  // p2p variant: no ghost rows, B = warps * rpw
        for (int r : {4, 2, 8, 1}) {
            if (B % r == 0 && B / r <= kResidentMaxWarps) {
                *ghost = 0;
                *rpw = r;
                *warps = B / r;
                return true;
            }
        }
        return false;
    }
    // ghost depth = steps between neighbour exchanges: the block depth, capped at
    // 8, the measured optimum (profiles/r1_sweep_1024_paths.jsonl: 4.04 vs 3.99
    // Tcell/s at G = 16; fewer redundant ghost rows against more exchanges)
    const int G = std::min(kResidentGhost, std::max(1, d->block_steps));
    if (B < G) return false;
    const int E = B + 2 * G;
    // a half-warp-wide lattice (W = 16, n = 512) packs two rows into each
    // register: +15% (profiles/r1_sweep_resident_pack.jsonl). Narrower ones
    // (n <= 256) measured slower packed: with so few rows per CTA the warps'
    // latency chains, not the lanes, are the limit.
    static constexpr int kPackedOrder[] = {2, 1, 3, 4};
    static constexpr int kWideOrder[] = {5, 4, 6, 3, 8, 2, 1};
    const int packed = d->W == 16 ? 2 : 1;
    for (int p : {packed, 1}) {
        const int* order = p > 1 ? kPackedOrder : kWideOrder;
        const int norder = p > 1 ? 4 : 7;
        for (int oi = 0; oi < norder; ++oi) {
            const int r = order[oi];
            if (E % (r * p) == 0 && E / (r * p) <= kResidentMaxWarps) {
                *ghost = G;
                *rpw = r;
                *warps = E / (r * p);
                *pack = p;
                return true;
            }
        }
        if (p == 1) break;
    }
    return false;
}

// Whether `cluster` CTAs of `threads` threads of `kern` can be co-scheduled
// (non-portable sizes > 8 enabled first). Memoised: the attribute and occupancy
// queries cost more host time than a short resident run.
bool cluster_launchable(ResidentKernel kern, int cluster, int threads) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<ResidentKernel, int>, bool>> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& kv : cache)
        if (kv.first.first == kern && kv.first.second == cluster) return kv.second;
    bool ok = true;
    if (cluster > 8 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        ok = false;
    if (ok) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(cluster));
        cfg.blockDim = dim3(static_cast<unsigned>(threads));
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int max_clusters = 0;
        ok = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) == cudaSuccess && max_clusters >= 1;
    }
    if (!ok) (void)cudaGetLastError();
    cache.emplace_back(std::make_pair(kern, cluster), ok);
    return ok;
}

// (single band only; with COUNT the kernels take the census after every step).
// Metrics of step s of this launch go to d->metrics[q * metrics_stride + metrics_base + s].
int launch_resident(bml_dev* d, long long steps, bool count, long long metrics_base, int metrics_stride,
                    bool* used) {
    *used = false;
    for (int cluster : {16, 8, 4, 2, 1}) {
        int G = 0, rpw = 0, nw = 0, pack = 1;
        if (!resident_plan(d, cluster, &G, &rpw, &nw, &pack)) continue;
        ResidentKernel kern = d->resident == 2
                                  ? (count ? pick_p2p<true>(rpw) : pick_p2p<false>(rpw))
                                  : (count ? pick_resident<true>(rpw, pack) : pick_resident<false>(rpw, pack));
        if (!kern || !cluster_launchable(kern, cluster, 32 * nw)) continue;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(cluster));
        cfg.blockDim = dim3(static_cast<unsigned>(32 * nw));
        cfg.dynamicSmemBytes = 0;
        cfg.stream = d->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        ResidentArgs ra{};
        ra.one = 1u;
        ra.src = d->row0(d->cur);
        ra.dst = d->row0(d->cur ^ 1);
        ra.n = d->n;
        ra.W = d->W;
        ra.pitch = d->pitch;
        ra.ghost = G;
        ra.steps = steps;
        ra.metrics = d->metrics ? d->metrics + metrics_base : nullptr;
        ra.metrics_stride = metrics_stride;
        ra.error_flag = d->err + 1;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (d->timing) {
            e0 = take_event(d);
            e1 = take_event(d);
            cudaEventRecord(e0, d->stream);
        }
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ra);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            if (d->timing) {
                d->ev_pool.push_back(e0);
                d->ev_pool.push_back(e1);
            }
            continue;
        }
        if (d->timing) {
            cudaEventRecord(e1, d->stream);
            d->pending.emplace_back(e0, e1);
        }
        ++d->launches;
        d->cur ^= 1;
        d->resident_cluster = cluster;
        d->kernel_steps[BML_KERNEL_RESIDENT] += steps;
        *used = true;
        return BML_OK;
    }
    return BML_OK;
}

}  // namespace

// ================================================================ C-ABI
extern "C" {

const char* bml_dev_last_error(void) { return g_last_error.c_str(); }

const char* bml_dev_version(void) { return "bml_dev 0.1.0 sm_100a bitplane-temporal"; }

int bml_dev_device_count(int* count) {
    if (!count) return fail(BML_EINVAL, "bml_dev_device_count: null pointer");
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
        (void)cudaGetLastError();
        *count = 0;
        return BML_OK;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    return BML_OK;
}

int bml_dev_create(int n, int device, bml_dev** out) {
    return create_common(n, 0, n, device, out);
}

int bml_dev_create_band(int n, int row_begin, int row_end, int device, bml_dev** out) {
    if (row_end - row_begin < kHalo && !(row_begin == 0 && row_end == n))
        return fail(BML_EINVAL, "bml_dev_create_band: a band needs >= 16 rows");
    return create_common(n, row_begin, row_end, device, out);
}

int bml_dev_destroy(bml_dev* d) {
    if (!d) return BML_OK;
    cudaSetDevice(d->device);
    if (d->stream) cudaStreamSynchronize(d->stream);
    if (d->own_stream && d->own_stream != d->stream) cudaStreamSynchronize(d->own_stream);
    for (void* p : d->ipc_opened) cudaIpcCloseMemHandle(p);
    for (int p = 0; p < 2; ++p) cudaFree(d->buf[p]);
    cudaFree(d->staging);
    cudaFree(d->scratch);
    cudaFree(d->err);
    if (d->err_host) cudaFreeHost(d->err_host);
    cudaFree(d->flags);
    cudaFree(d->metrics);
    for (auto& pr : d->pending) {
        d->ev_pool.push_back(pr.first);
        d->ev_pool.push_back(pr.second);
    }
    for (cudaEvent_t e : d->ev_pool) cudaEventDestroy(e);
    if (d->own_stream) cudaStreamDestroy(d->own_stream);
    delete d;
    return BML_OK;
}

int bml_dev_set_stream(bml_dev* d, void* stream) {
    if (int rc = check(d)) return rc;
    cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : d->own_stream;
    if (next != d->stream) {
        // order the work already queued on the old stream before the new one's
        cudaEvent_t ev = take_event(d);
        if (!ev) return fail(BML_ECUDA, "bml_dev_set_stream: cudaEventCreate failed");
        cudaError_t e = cudaEventRecord(ev, d->stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(next, ev, 0);
        d->ev_pool.push_back(ev);  // reusable: the wait captured the recorded work
        if (e != cudaSuccess) return cuda_fail(e, "bml_dev_set_stream");
    }
    d->stream = next;
    return BML_OK;
}

int bml_dev_sync(bml_dev* d) {
    if (int rc = check(d)) return rc;
    BML_CUDA(cudaStreamSynchronize(d->stream));
    return check_errors(d);
}

int bml_dev_configure(bml_dev* d, int block_steps, int strip_rows) {
    if (int rc = check(d)) return rc;
    if (block_steps) {
        if (block_steps != 1 && block_steps != 2 && block_steps != 4 && block_steps != 8 &&
            block_steps != 16)
            return fail(BML_EINVAL, "block_steps must be one of 1, 2, 4, 8, 16");
        d->block_steps = block_steps;
    }
    if (strip_rows) {
        if (strip_rows < -65536 || strip_rows > 65536)
            return fail(BML_EINVAL, "strip_rows must be in [1, 65536], -1 (auto) or -ns (ns >= 2 strips)");
        if (strip_rows == -1) strip_rows = 0;
        if (d->connected && strip_rows > 0 && strip_rows < kHalo)
            return fail(BML_EINVAL, "connected bands need strip_rows >= 16");
        d->strip_rows = strip_rows;
    }
    return BML_OK;
}

int bml_dev_set_resident(bml_dev* d, int mode) {
    if (int rc = check(d)) return rc;
    if (mode < 0 || mode > 2) return fail(BML_EINVAL, "bml_dev_set_resident: mode must be 0, 1 or 2");
    d->resident = mode;
    return BML_OK;
}

int bml_dev_set_variant(bml_dev* d, int variant) {
    if (int rc = check(d)) return rc;
    if (variant < 0 || variant > 6) return fail(BML_EINVAL, "bml_dev_set_variant: 0 (auto) .. 6");
    if (d->connected)
        return fail(BML_EINVAL, "bml_dev_set_variant: set before bml_dev_connect (all bands alike)");
    d->variant = variant;
    std::fill(std::begin(d->ns_cache_k), std::end(d->ns_cache_k), 0);
    return BML_OK;
}

int bml_dev_path(bml_dev* d, int* resident_cluster) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    if (resident_cluster) *resident_cluster = d->resident_cluster;
    return BML_OK;
}

int bml_dev_last_kernel(bml_dev* d, int* kernel, int64_t* steps) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    int best = BML_KERNEL_NONE;
    for (int k = 1; k < 6; ++k)
        if (d->kernel_steps[k] > d->kernel_steps[best]) best = k;
    if (kernel) *kernel = best;
    if (steps) *steps = d->kernel_steps[best];
    return BML_OK;
}

int bml_dev_last_launch(bml_dev* d, int* nstrips, int* items, int* grid) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    if (nstrips) *nstrips = d->last_nstrips;
    if (items) *items = d->last_items;
    if (grid) *grid = d->last_grid;
    return BML_OK;
}

int bml_dev_last_kernel_launch(bml_dev* d, int* nstrips, int* items, int* grid) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    int kind = BML_KERNEL_NONE;
    if (int rc = bml_dev_last_kernel(d, &kind, nullptr)) return rc;
    const bool streaming = kind != BML_KERNEL_NONE && kind != BML_KERNEL_RESIDENT;
    if (nstrips) *nstrips = streaming ? d->kind_geom[kind][0] : 0;
    if (items) *items = streaming ? d->kind_geom[kind][1] : 0;
    if (grid) *grid = streaming ? d->kind_geom[kind][2] : 0;
    return BML_OK;
}

int bml_dev_info(bml_dev* d, int* n, int* row_begin, int* row_end, int* block_steps,
                 int* strip_rows, size_t* device_bytes) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    if (n) *n = d->n;
    if (row_begin) *row_begin = d->row_begin;
    if (row_end) *row_end = d->row_end;
    if (block_steps) *block_steps = d->block_steps;
    if (strip_rows) *strip_rows = d->strip_rows;
    if (device_bytes)
        *device_bytes = 2 * static_cast<size_t>(d->rows + 2 * kHalo) * d->pitch * sizeof(uint2) +
                        static_cast<size_t>(d->rows) * d->n;
    return BML_OK;
}

int bml_dev_enable_timing(bml_dev* d, int enable) {
    if (int rc = check(d)) return rc;
    d->timing = enable != 0;
    return BML_OK;
}

int bml_dev_kernel_stats(bml_dev* d, int64_t* launches, double* kernel_ms, int reset) {
    if (int rc = check(d)) return rc;
    BML_CUDA(cudaStreamSynchronize(d->stream));
    harvest_timing(d);
    if (launches) *launches = d->launches;
    if (kernel_ms) *kernel_ms = d->kernel_ms;
    if (reset) {
        d->launches = 0;
        d->kernel_ms = 0.0;
    }
    return BML_OK;
}

namespace {

// H2D into the staging rows, then bit-pack (and the single band's ghost-row
// images), all enqueued on the handle's stream. Invalid cells set err[0].
int enqueue_upload(bml_dev* d, const uint8_t* src, size_t src_pitch, const char* who) {
    if (!src) return fail(BML_EINVAL, std::string(who) + ": src is null");
    if (src_pitch < static_cast<size_t>(d->n)) return fail(BML_EINVAL, std::string(who) + ": pitch smaller than a row");
    BML_CUDA(cudaMemsetAsync(d->err, 0, sizeof(int), d->stream));
    BML_CUDA(cudaMemcpy2DAsync(d->staging, d->n, src, src_pitch, d->n, d->rows, cudaMemcpyDefault, d->stream));
    const long long total = static_cast<long long>(d->rows) * d->W;
    pack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, d->stream>>>(
        d->staging, d->n, d->row0(d->cur), d->n, d->W, d->pitch, d->rows, d->err);
    BML_CUDA(cudaGetLastError());
    if (d->single_band()) {
        if (int rc = fill_images(d, d->cur)) return rc;
    }
    return BML_OK;
}

int enqueue_download(bml_dev* d, uint8_t* dst, size_t dst_pitch, const char* who) {
    if (!dst) return fail(BML_EINVAL, std::string(who) + ": dst is null");
    if (dst_pitch < static_cast<size_t>(d->n)) return fail(BML_EINVAL, std::string(who) + ": pitch smaller than a row");
    const long long total = static_cast<long long>(d->rows) * d->W;
    unpack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, d->stream>>>(
        d->row0(d->cur), d->staging, d->n, d->n, d->W, d->pitch, d->rows);
    BML_CUDA(cudaGetLastError());
    BML_CUDA(cudaMemcpy2DAsync(dst, dst_pitch, d->staging, d->n, d->n, d->rows, cudaMemcpyDefault, d->stream));
    return BML_OK;
}

}  // namespace

int bml_dev_upload(bml_dev* d, const uint8_t* src, size_t src_pitch) {
    const NvtxRange nvtx_range("bml_dev_upload");
    if (int rc = check(d)) return rc;
    if (int rc = enqueue_upload(d, src, src_pitch, "bml_dev_upload")) return rc;
    BML_CUDA(enqueue_error_readback(d));
    BML_CUDA(cudaStreamSynchronize(d->stream));
    if (d->err_host[0]) {
        cudaMemsetAsync(d->err, 0, sizeof(int), d->stream);
        return fail(BML_EINVAL, "bml_dev_upload: cell value outside {0,1,2}");
    }
    return errors_after_sync(d);
}

int bml_dev_download(bml_dev* d, uint8_t* dst, size_t dst_pitch) {
    const NvtxRange nvtx_range("bml_dev_download");
    if (int rc = check(d)) return rc;
    if (int rc = enqueue_download(d, dst, dst_pitch, "bml_dev_download")) return rc;
    BML_CUDA(enqueue_error_readback(d));  // one synchronisation for data and flags
    BML_CUDA(cudaStreamSynchronize(d->stream));
    return errors_after_sync(d);
}

int bml_dev_upload_async(bml_dev* d, const uint8_t* src, size_t src_pitch) {
    const NvtxRange nvtx_range("bml_dev_upload_async");
    if (int rc = check(d)) return rc;
    return enqueue_upload(d, src, src_pitch, "bml_dev_upload_async");
}

int bml_dev_download_async(bml_dev* d, uint8_t* dst, size_t dst_pitch) {
    const NvtxRange nvtx_range("bml_dev_download_async");
    if (int rc = check(d)) return rc;
    return enqueue_download(d, dst, dst_pitch, "bml_dev_download_async");
}

int bml_dev_init_random_masked(bml_dev* d, double rho, uint64_t seed, uint64_t reject_mask) {
    const NvtxRange nvtx_range("bml_dev_init_random");
    if (int rc = check(d)) return rc;
    if (!(rho >= 0.0 && rho <= 1.0))
        return fail(BML_EINVAL, "init_grid: density must be in [0, 1]");
    if (static_cast<unsigned long long>(d->n) * d->n > (1ull << 32))
        return fail(BML_EINVAL, "bml_dev_init_random: device init supports n <= 65536");
    std::string msg;
    const int rc = bml_init::init_planes(d->row0(d->cur), d->pitch, d->n, d->row_begin,
                                         d->row_end, rho, seed, reject_mask, d->stream, d->sms,
                                         &msg);
    if (rc == 3) return fail(BML_ENOMEM, "bml_dev_init_random: " + msg);
    if (rc != 0) return fail(BML_ECUDA, "bml_dev_init_random: " + msg);
    if (d->single_band()) {
        if (int r2 = fill_images(d, d->cur)) return r2;
    }
    BML_CUDA(cudaStreamSynchronize(d->stream));
    return BML_OK;
}

int bml_dev_init_random(bml_dev* d, double rho, uint64_t seed) {
    return bml_dev_init_random_masked(d, rho, seed, 0);
}

int bml_dev_encode_ppm(bml_dev* d, uint8_t* dst, size_t dst_pitch) {
    if (int rc = check(d)) return rc;
    if (!dst) return fail(BML_EINVAL, "bml_dev_encode_ppm: dst is null");
    const size_t row_bytes = 3 * static_cast<size_t>(d->n);
    if (dst_pitch < row_bytes) return fail(BML_EINVAL, "bml_dev_encode_ppm: pitch smaller than a row");
    uint8_t* rgb = nullptr;
    BML_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rgb), row_bytes * d->rows, d->stream));
    const long long total = static_cast<long long>(d->rows) * d->W;
    ppm_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, d->stream>>>(
        d->row0(d->cur), rgb, static_cast<long long>(row_bytes), d->n, d->W, d->pitch, d->rows);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(dst, dst_pitch, rgb, row_bytes, row_bytes, d->rows, cudaMemcpyDefault,
                              d->stream);
    cudaFreeAsync(rgb, d->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream);
    if (e != cudaSuccess) return cuda_fail(e, "bml_dev_encode_ppm");
    return BML_OK;
}

int bml_dev_digest_segment(bml_dev* d, uint64_t seg[6]) {
    const NvtxRange nvtx_range("bml_dev_digest_segment");
    if (int rc = check(d)) return rc;
    if (!seg) return fail(BML_EINVAL, "bml_dev_digest_segment: seg is null");
    std::string msg;
    const int rc = bml_digest::segment(d->row0(d->cur), d->n, d->W, d->pitch, d->rows, d->stream,
                                       d->sms, seg, &msg);
    if (rc == 3) return fail(BML_ENOMEM, msg);
    if (rc != 0) return fail(BML_ECUDA, msg);
    return BML_OK;
}

int bml_dev_digest(bml_dev* d, uint64_t* digest) {
    if (int rc = check(d)) return rc;
    if (!digest) return fail(BML_EINVAL, "bml_dev_digest: digest is null");
    if (!d->single_band())
        return fail(BML_EINVAL, "bml_dev_digest: a row band hashes only its rows; combine "
                                "bml_dev_digest_segment() of all bands with bml_digest_finish()");
    uint64_t seg[6];
    if (int rc = bml_dev_digest_segment(d, seg)) return rc;
    *digest = bml_digest::finish(seg, 1);
    return BML_OK;
}

int bml_digest_finish(const uint64_t* segs, int count, uint64_t* digest) {
    if (!digest || count < 0 || (count > 0 && !segs))
        return fail(BML_EINVAL, "bml_digest_finish: bad arguments");
    *digest = bml_digest::finish(segs, count);
    return BML_OK;
}

int bml_dev_counts(bml_dev* d, int64_t* lr, int64_t* tb) {
    const NvtxRange nvtx_range("bml_dev_counts");
    if (int rc = check(d)) return rc;
    BML_CUDA(cudaMemsetAsync(d->scratch, 0, 2 * sizeof(unsigned long long), d->stream));
    counts_kernel<<<d->sms * 4, 256, 0, d->stream>>>(d->row0(d->cur), d->W, d->pitch, d->rows,
                                                     d->scratch);
    BML_CUDA(cudaGetLastError());
    unsigned long long h[2];
    BML_CUDA(cudaMemcpyAsync(h, d->scratch, sizeof h, cudaMemcpyDeviceToHost, d->stream));
    BML_CUDA(cudaStreamSynchronize(d->stream));
    if (lr) *lr = static_cast<int64_t>(h[0]);
    if (tb) *tb = static_cast<int64_t>(h[1]);
    return BML_OK;
}

int bml_dev_phase(bml_dev* d, int phase, int64_t* moved) {
    if (int rc = check(d)) return rc;
    if (phase != BML_PHASE_HORIZONTAL && phase != BML_PHASE_VERTICAL)
        return fail(BML_EINVAL, "bml_dev_phase: phase must be 0 (horizontal) or 1 (vertical)");
    if (!d->single_band())
        return fail(BML_EINVAL, "bml_dev_phase: single phases need a single-band handle");
    BML_CUDA(cudaMemsetAsync(d->scratch, 0, sizeof(unsigned long long), d->stream));
    PhaseArgs a{};
    a.src = d->row0(d->cur);
    a.dst = d->row0(d->cur ^ 1);
    a.n = d->n;
    a.W = d->W;
    a.pitch = d->pitch;
    a.rows = d->rows;
    a.last_mask = d->last_mask;
    a.moved = d->scratch;
    const long long total = static_cast<long long>(d->rows) * d->W;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    if (phase == BML_PHASE_HORIZONTAL)
        phase_h_kernel<<<grid, 256, 0, d->stream>>>(a);
    else
        phase_v_kernel<<<grid, 256, 0, d->stream>>>(a);
    BML_CUDA(cudaGetLastError());
    d->cur ^= 1;
    if (moved) {
        unsigned long long h = 0;
        BML_CUDA(cudaMemcpyAsync(&h, d->scratch, sizeof h, cudaMemcpyDeviceToHost, d->stream));
        BML_CUDA(cudaStreamSynchronize(d->stream));
        *moved = static_cast<int64_t>(h);
    }
    return BML_OK;
}

int bml_dev_set_census(bml_dev* d, int every_step) {
    if (int rc = check(d)) return rc;
    if (every_step != 0 && every_step != 1) return fail(BML_EINVAL, "bml_dev_set_census: 0 or 1");
    d->census_every_step = every_step;
    return BML_OK;
}

int bml_dev_debug_fault(bml_dev* d, int64_t at_step, int row, int col) {
    if (int rc = check(d)) return rc;
    if (!d->single_band()) return fail(BML_EINVAL, "bml_dev_debug_fault: single-band handles only");
    if (at_step < 0 || row < 0 || row >= d->rows || col < 0 || col >= d->n)
        return fail(BML_EINVAL, "bml_dev_debug_fault: step/row/col out of range");
    if (d->faults.size() >= 8) return fail(BML_EINVAL, "bml_dev_debug_fault: at most 8 armed faults");
    d->faults.push_back({at_step, row, col});
    return BML_OK;
}

namespace {

// In-place layout conversion of the current buffer (to or from the even/odd
// layout). A single band converts its rows and ghost rows in one pass; a
// connected band converts its own rows, then its ghost rows once both
// neighbours have published every launch so far (their last launch wrote them).
int eo_convert(bml_dev* d, bool to_eo) {
    const int pairs = d->W / 2;
    const long long rows_total = d->connected ? d->rows : d->rows + 2 * kHalo;
    uint2* base = d->connected ? d->row0(d->cur) : d->buf[d->cur];
    const unsigned blocks = static_cast<unsigned>((rows_total * pairs + 255) / 256);
    if (to_eo)
        eo_convert_kernel<true><<<blocks, 256, 0, d->stream>>>(base, rows_total, d->pitch, pairs);
    else
        eo_convert_kernel<false><<<blocks, 256, 0, d->stream>>>(base, rows_total, d->pitch, pairs);
    BML_CUDA(cudaGetLastError());
    if (d->connected) {
        const dim3 g(static_cast<unsigned>((kHalo * pairs + 255) / 256), 2);
        if (to_eo)
            eo_convert_ghost_kernel<true><<<g, 256, 0, d->stream>>>(d->row0(d->cur), d->pitch, pairs, d->rows,
                                                                    d->flags, d->flags + 1, d->pub_sum, d->err + 1);
        else
            eo_convert_ghost_kernel<false><<<g, 256, 0, d->stream>>>(d->row0(d->cur), d->pitch, pairs, d->rows,
                                                                     d->flags, d->flags + 1, d->pub_sum, d->err + 1);
        BML_CUDA(cudaGetLastError());
    }
    return BML_OK;
}

// `seg` steps from step `from` of the current call: the resident kernel when the
// lattice qualifies, else streaming launches of <= block_steps steps. `measured`
// marks the steps whose census the kernels took.
int run_segment(bml_dev* d, long long from, long long seg, bool count, bool every, int stride,
                std::vector<char>& measured) {
    bool resident_used = false;
    if (int rc = launch_resident(d, seg, count, from, stride, &resident_used)) return rc;
    if (resident_used) {
        if (count) std::fill(measured.begin() + from, measured.begin() + from + seg, 1);
        return BML_OK;
    }
    const int metrics = count ? (every ? 2 : 1) : 0;
    long long done = 0;
    if (d->use_eo() && d->block_steps == 16 && seg >= kEoMinSteps) {
        // even/odd layout for the whole 14-step (12 with metrics) blocks of the
        // run: convert the current buffer in place, step, convert back
        if (int rc = eo_convert(d, true)) return rc;
        d->eo_active = true;
        const int ek = d->eo_depth(metrics);
        for (; seg - done >= ek; done += ek) {
            if (int rc = launch_block(d, ek, count, every, static_cast<int>(from + done), stride)) {
                d->eo_active = false;
                eo_convert(d, false);  // leave the buffer in the standard layout
                return rc;
            }
            if (count) {
                if (every)
                    std::fill(measured.begin() + from + done, measured.begin() + from + done + ek, 1);
                else
                    measured[from + done + ek - 1] = 1;
            }
        }
        d->eo_active = false;
        if (int rc = eo_convert(d, false)) return rc;
    }
    const int wk = d->use_wide() && d->block_steps == 16 ? d->wide_depth(metrics) : 0;
    for (; done < seg;) {
        const int k = (wk && seg - done >= wk) ? wk : largest_block_at_most(seg - done, d->block_steps);
        if (int rc = launch_block(d, k, count, every, static_cast<int>(from + done), stride)) return rc;
        if (count) {
            if (every)
                std::fill(measured.begin() + from + done, measured.begin() + from + done + k, 1);
            else
                measured[from + done + k - 1] = 1;  // COUNT 1: census after the launch's last step
        }
        done += k;
    }
    return BML_OK;
}

}  // namespace

int bml_dev_step(bml_dev* d, int64_t steps, int64_t* lr_moved, int64_t* tb_moved,
                 int64_t* lr_count, int64_t* tb_count) {
    const NvtxRange nvtx_range("bml_dev_step");
    if (int rc = check(d)) return rc;
    if (steps < 0) return fail(BML_EINVAL, "bml_dev_step: steps must be >= 0");
    if (!d->single_band() && !d->connected)
        return fail(BML_EINVAL, "bml_dev_step: a partial row band must be connected (bml_dev_connect) "
                                "before stepping");
    std::vector<bml_dev::Fault> faults;
    faults.swap(d->faults);  // armed for this call only
    std::stable_sort(faults.begin(), faults.end(),
                     [](const bml_dev::Fault& x, const bml_dev::Fault& y) { return x.at < y.at; });
    if (steps == 0 && faults.empty()) return BML_OK;
    const bool count = lr_moved || tb_moved || lr_count || tb_count;
    if (count && steps > (1LL << 26))
        return fail(BML_EINVAL, "bml_dev_step: at most 2^26 steps per call with metrics");
    // Vehicle census (the reference's count_vehicles after every step,
    // engine.cpp:219-224), measured in the kernels: row bands and strict mode
    // after every step (COUNT 2), a single band otherwise after each launch's
    // last step (COUNT 1; the resident kernel always per step).
    const bool want_counts = lr_count || tb_count;
    const bool banded = !d->single_band();
    const bool every = want_counts && (banded || d->census_every_step);
    int64_t lr0 = 0, tb0 = 0;
    if (want_counts && !banded) {
        if (int rc = bml_dev_counts(d, &lr0, &tb0)) return rc;
    }
    if (count) {
        if (int rc = ensure_metrics(d, steps)) return rc;
        BML_CUDA(cudaMemsetAsync(d->metrics, 0, 4 * steps * sizeof(unsigned long long), d->stream));
    }
    std::vector<char> measured(count ? static_cast<size_t>(steps) : 0, 0);
    d->resident_cluster = 0;
    std::fill(std::begin(d->kernel_steps), std::end(d->kernel_steps), 0LL);
    const int stride = static_cast<int>(steps);
    long long done = 0;
    size_t fi = 0;
    for (;;) {
        for (; fi < faults.size() && faults[fi].at <= done; ++fi) {  // injected faults due now
            if (faults[fi].at > steps) continue;
            debug_toggle_kernel<<<1, 32, 0, d->stream>>>(d->row0(d->cur), d->pitch, faults[fi].row,
                                                         faults[fi].col);
            BML_CUDA(cudaGetLastError());
            if (int rc = fill_images(d, d->cur)) return rc;
        }
        if (done >= steps) break;
        long long seg_end = steps;
        if (fi < faults.size() && faults[fi].at < steps) seg_end = faults[fi].at;
        if (int rc = run_segment(d, done, seg_end - done, count, every, stride, measured)) return rc;
        done = seg_end;
    }
    if (!count) return BML_OK;
    std::vector<unsigned long long> h(static_cast<size_t>(4 * steps));
    BML_CUDA(cudaMemcpyAsync(h.data(), d->metrics, h.size() * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, d->stream));
    BML_CUDA(cudaStreamSynchronize(d->stream));
    if (int rc = check_errors(d)) return rc;
    int64_t lc = lr0, tc = tb0;
    long long violated = -1;
    for (int64_t s = 0; s < steps; ++s) {
        if (measured[s]) {
            lc = static_cast<int64_t>(h[2 * steps + s]);
            tc = static_cast<int64_t>(h[3 * steps + s]);
            if (want_counts && !banded && violated < 0 && (lc != lr0 || tc != tb0)) violated = s;
        }
        if (lr_moved) lr_moved[s] = static_cast<int64_t>(h[s]);
        if (tb_moved) tb_moved[s] = static_cast<int64_t>(h[steps + s]);
        if (lr_count) lr_count[s] = lc;
        if (tb_count) tb_count[s] = tc;
    }
    if (violated >= 0) {
        const int64_t vl = static_cast<int64_t>(h[2 * steps + violated]);
        const int64_t vt = static_cast<int64_t>(h[3 * steps + violated]);
        return fail(BML_ECONSERVE, "conservation violated at step " + std::to_string(violated + 1) + " of " +
                                       std::to_string(steps) + ": lr " + std::to_string(vl) + "/" +
                                       std::to_string(lr0) + ", tb " + std::to_string(vt) + "/" +
                                       std::to_string(tb0));
    }
    return BML_OK;
}

// ---------------------------------------------------------------- multi-band
int bml_dev_export(bml_dev* d, void* blob, size_t* size) {
    if (int rc = check(d)) return rc;
    if (!blob || !size || *size < sizeof(IpcBlob))
        return fail(BML_EINVAL, "bml_dev_export: blob buffer too small");
    IpcBlob b{};
    b.magic = kBlobMagic;
    b.n = d->n;
    b.row_begin = d->row_begin;
    b.row_end = d->row_end;
    b.pitch = d->pitch;
    b.W = d->W;
    b.device = d->device;
    for (int p = 0; p < 2; ++p) BML_CUDA(cudaIpcGetMemHandle(&b.buf[p], d->buf[p]));
    BML_CUDA(cudaIpcGetMemHandle(&b.flags, d->flags));
    std::memcpy(blob, &b, sizeof b);
    *size = sizeof b;
    return BML_OK;
}

namespace {

int link_peer(bml_dev* d, uint2* const peer_buf[2], unsigned long long* peer_flags, int peer_rows,
              bool is_up) {
    for (int p = 0; p < 2; ++p) {
        uint2* peer_row0 = peer_buf[p] + static_cast<long long>(kHalo) * d->pitch;
        if (is_up)
            d->up_halo[p] = peer_row0 + static_cast<long long>(peer_rows) * d->pitch;  // its bottom ghosts
        else
            d->down_halo[p] = peer_row0;  // row (r - rows) in [-kHalo, 0): its top ghosts
    }
    if (is_up)
        d->up_flag = peer_flags + 1;  // the neighbour above waits on its bottom flag
    else
        d->down_flag = peer_flags;  // the neighbour below waits on its top flag
    return BML_OK;
}

int validate_neighbours(bml_dev* d, int up_end, int up_n, int up_pitch, int dn_begin, int dn_n,
                        int dn_pitch) {
    if (up_n != d->n || dn_n != d->n || up_pitch != d->pitch || dn_pitch != d->pitch)
        return fail(BML_EINVAL, "bml_dev_connect: neighbour lattice geometry differs");
    if (up_end % d->n != d->row_begin)
        return fail(BML_EINVAL, "bml_dev_connect: up neighbour does not end where this band begins");
    if (dn_begin != d->row_end % d->n)
        return fail(BML_EINVAL, "bml_dev_connect: down neighbour does not begin where this band ends");
    if (d->strip_rows > 0 && d->strip_rows < kHalo) d->strip_rows = kHalo;
    return BML_OK;
}

}  // namespace

int bml_dev_connect(bml_dev* d, const void* up_blob, const void* down_blob) {
    if (int rc = check(d)) return rc;
    if (!up_blob || !down_blob) return fail(BML_EINVAL, "bml_dev_connect: null blob");
    IpcBlob up, dn;
    std::memcpy(&up, up_blob, sizeof up);
    std::memcpy(&dn, down_blob, sizeof dn);
    if (up.magic != kBlobMagic || dn.magic != kBlobMagic)
        return fail(BML_EINVAL, "bml_dev_connect: not a bml_dev export blob");
    if (int rc = validate_neighbours(d, up.row_end, up.n, up.pitch, dn.row_begin, dn.n, dn.pitch))
        return rc;
    const bool same = std::memcmp(&up.buf[0], &dn.buf[0], sizeof(cudaIpcMemHandle_t)) == 0;
    auto open = [&](const cudaIpcMemHandle_t& h, void** p) -> int {
        cudaError_t e = cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
        d->ipc_opened.push_back(*p);
        return BML_OK;
    };
    void *ub[2], *uf, *db[2], *df;
    for (int p = 0; p < 2; ++p)
        if (int rc = open(up.buf[p], &ub[p])) return rc;
    if (int rc = open(up.flags, &uf)) return rc;
    if (same) {
        db[0] = ub[0];
        db[1] = ub[1];
        df = uf;
    } else {
        for (int p = 0; p < 2; ++p)
            if (int rc = open(dn.buf[p], &db[p])) return rc;
        if (int rc = open(dn.flags, &df)) return rc;
    }
    uint2* ubp[2] = {static_cast<uint2*>(ub[0]), static_cast<uint2*>(ub[1])};
    uint2* dbp[2] = {static_cast<uint2*>(db[0]), static_cast<uint2*>(db[1])};
    link_peer(d, ubp, static_cast<unsigned long long*>(uf), up.row_end - up.row_begin, true);
    link_peer(d, dbp, static_cast<unsigned long long*>(df), dn.row_end - dn.row_begin, false);
    d->connected = true;
    std::fill(std::begin(d->ns_cache_k), std::end(d->ns_cache_k), 0);  // strip limits changed
    return BML_OK;
}

int bml_dev_connect_local(bml_dev* d, bml_dev* up, bml_dev* down) {
    if (int rc = check(d)) return rc;
    if (!up || !down) return fail(BML_EINVAL, "bml_dev_connect_local: null neighbour");
    if (int rc = validate_neighbours(d, up->row_end, up->n, up->pitch, down->row_begin, down->n,
                                     down->pitch))
        return rc;
    for (bml_dev* peer : {up, down}) {
        if (peer->device != d->device) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, d->device, peer->device);
            if (!can) return fail(BML_ECUDA, "bml_dev_connect_local: no peer access between devices");
            cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return cuda_fail(e, "cudaDeviceEnablePeerAccess");
            (void)cudaGetLastError();
        }
    }
    link_peer(d, up->buf, up->flags, up->rows, true);
    link_peer(d, down->buf, down->flags, down->rows, false);
    d->connected = true;
    std::fill(std::begin(d->ns_cache_k), std::end(d->ns_cache_k), 0);  // strip limits changed
    return BML_OK;
}

int bml_dev_exchange_halos(bml_dev* d) {
    const NvtxRange nvtx_range("bml_dev_exchange_halos");
    if (int rc = check(d)) return rc;
    if (!d->connected && !d->single_band())
        return fail(BML_EINVAL, "bml_dev_exchange_halos: a partial row band must be connected first");
    if (!d->connected) return fill_images(d, d->cur);
    push_halo_kernel<<<1, 1024, 0, d->stream>>>(d->row0(d->cur), d->W, d->pitch, d->rows,
                                                d->up_halo[d->cur], d->down_halo[d->cur],
                                                d->up_flag, d->down_flag, d->ncols());
    BML_CUDA(cudaGetLastError());
    d->pub_sum += static_cast<unsigned long long>(d->ncols());
    return BML_OK;
}

}  // extern "C"
