/* include/bml_dev.h — C-ABI of the B200-native BML (Biham–Middleton–Levine) step.
 *
 * This is the drop-in boundary: the reference C++ API (namespace bml, SURVEY.md
 * §8(b)) is re-implemented on the host in paper_1804_07981_b200/csrc/host/ and
 * reaches the GPU only through these functions. Plain pointers and sizes, no
 * torch or C++ types. All functions return a status code:
 *
 *   BML_OK      0  success
 *   BML_EINVAL  1  invalid argument   (reference: std::invalid_argument)
 *   BML_ECUDA   2  CUDA / peer error  (reference: none — new failure mode)
 *   BML_ENOMEM  3  device allocation failed
 *   BML_ECONSERVE 4 per-step vehicle conservation violated
 *                   (reference: std::logic_error, src/engine.cpp:219-224)
 *
 * bml_dev_last_error() returns a thread-local message for the last failure.
 * A handle is not thread-safe; one host thread drives it.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj):
 *   bml_dev_create        GridPair make_grid_pair(Backend, const Grid&)   include/bml/engine.hpp:60
 *                         (allocation half: the device-resident double buffer)
 *   bml_dev_upload        make_grid_pair's interior copy                   src/engine.cpp:59-64, src/grid.cpp:37-49
 *   bml_dev_init_random   Grid init_grid(const SeedSpec&)                  include/bml/seeding.hpp:42
 *   bml_dev_phase         void step_phase(Backend, GridPair&, Phase, int)  include/bml/engine.hpp:66
 *   bml_dev_step          void step(Backend, GridPair&, int) x steps,      include/bml/engine.hpp:70
 *                         and the loops of Grid run(...)                   src/engine.cpp:206-235
 *                         with moved_in_phase / count_vehicles fused       src/metrics.cpp:8-29
 *   bml_dev_counts        VehicleCounts count_vehicles(const Grid&)        include/bml/metrics.hpp:20
 *   bml_dev_digest        std::uint64_t grid_digest(const Grid&)           include/bml/digest.hpp:23
 *   bml_dev_encode_ppm    std::vector<uint8_t> encode_ppm(const Grid&)     include/bml/snapshot.hpp:21
 *   bml_dev_download      readback: Grid::interior / data                  include/bml/grid.hpp:38-47
 *   bml_dev_destroy       ~GridPair
 *
 * Lattice bytes crossing this boundary use the reference cell encoding
 * (include/bml/cell.hpp:9): 0 = Empty, 1 = LR, 2 = TB. On the device the
 * lattice is bit-sliced (two bit planes, 32 cells per word); see DESIGN.md.
 */
#ifndef BML_DEV_H
#define BML_DEV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BML_OK 0
#define BML_EINVAL 1
#define BML_ECUDA 2
#define BML_ENOMEM 3
#define BML_ECONSERVE 4

#define BML_PHASE_HORIZONTAL 0 /* bml::Phase::Horizontal — LR vehicles move right */
#define BML_PHASE_VERTICAL 1   /* bml::Phase::Vertical   — TB vehicles move down  */

typedef struct bml_dev bml_dev;

/* Number of visible CUDA devices. */
int bml_dev_device_count(int *count);

/* Allocate a device-resident n x n torus on CUDA device `device` (-1 = the
 * calling thread's current device); the whole lattice is one row band. */
int bml_dev_create(int n, int device, bml_dev **out);

/* Allocate rows [row_begin, row_end) of an n x n torus as one row band on
 * `device` (multi-GPU decomposition). The band exchanges
 * halo rows with its two neighbours after bml_dev_connect(). */
int bml_dev_create_band(int n, int row_begin, int row_end, int device, bml_dev **out);

int bml_dev_destroy(bml_dev *dev);

/* Copy the band's rows in from host (or device) memory: `src` points at cell
 * (row_begin, 0); consecutive rows are `src_pitch` bytes apart. A halo-layout
 * reference Grid passes data()+stride+1 with pitch n+2. Cells must be 0/1/2. */
int bml_dev_upload(bml_dev *dev, const uint8_t *src, size_t src_pitch);

/* Copy the band's rows out, same addressing as bml_dev_upload. */
int bml_dev_download(bml_dev *dev, uint8_t *dst, size_t dst_pitch);

/* Fill the band's rows exactly as the reference init_grid({n, rho, seed})
 * does (SplitMix64 + descending Fisher–Yates, src/seeding.cpp:11-51), computed
 * on the device: parallel counter-based draws with a rejection fix-up, a
 * stable sort of the swap targets, and chain resolution of the swaps (see
 * csrc/bml_init.cu). n <= 65536. Needs 16·n² bytes of temporary device memory
 * (64 GiB at n = 65536), released before returning. Connected bands call
 * bml_dev_exchange_halos() afterwards, as after an upload. */
int bml_dev_init_random(bml_dev *dev, double rho, uint64_t seed);

/* TEST HOOK (not a reference interface): as bml_dev_init_random, but a draw r
 * with (r & reject_mask) == 0 is rejected as well, which drives the rejection
 * fix-up path at small n. reject_mask = 0 is exactly bml_dev_init_random. */
int bml_dev_init_random_masked(bml_dev *dev, double rho, uint64_t seed, uint64_t reject_mask);

/* Asynchronous forms: the same copies and (un)packing, enqueued on the handle's
 * stream without waiting. `src` / `dst` must stay valid (pinned host memory for
 * real overlap) until bml_dev_sync(), which also reports an invalid cell of an
 * asynchronous upload (BML_EINVAL). With bml_dev_step (no metrics, also
 * asynchronous) this lets a caller overlap one lattice's transfers with another
 * handle's stepping; bench.py's e2e leg pipelines two handles this way. */
int bml_dev_upload_async(bml_dev *dev, const uint8_t *src, size_t src_pitch);
int bml_dev_download_async(bml_dev *dev, uint8_t *dst, size_t dst_pitch);

/* One phase (step_phase). `moved` (nullable) receives the vehicles that
 * advanced (moved_in_phase). Single-band handles only. */
int bml_dev_phase(bml_dev *dev, int phase, int64_t *moved);

/* `steps` full steps (LR phase then TB phase each). Each of the four metric
 * arrays is nullable; when any is non-NULL, all requested arrays (length
 * `steps`) receive the per-step values of the reference observer loop
 * (engine.cpp:211-235): lr_moved, tb_moved, and the post-step lr/tb counts.
 * The moved counts are popcounts fused into the step kernels. The vehicle
 * census (count_vehicles after a step, engine.cpp:219-224) is measured inside
 * the kernels too:
 *   - row bands (counts change as TB vehicles cross band edges), the
 *     cluster-resident small-lattice kernel, and strict mode
 *     (bml_dev_set_census(dev, 1)): after EVERY step;
 *   - otherwise (single band, streaming kernel): after the last step of every
 *     launch (every <= 16 steps); in between, the last measured count.
 * A single band checks every measured census against the counts before the
 * run. On a difference the arrays are still filled (through the violating
 * step) and BML_ECONSERVE is returned; the message names the first step, 1-based
 * within this call, whose census differs — the exact step the reference would
 * throw at when the census is per step, else the launch boundary that saw it. */
int bml_dev_step(bml_dev *dev, int64_t steps, int64_t *lr_moved, int64_t *tb_moved,
                 int64_t *lr_count, int64_t *tb_count);

/* grid_digest (FNV-1a-64 over the cells, row-major; src/digest.cpp:5-14),
 * computed on the device, bit-identical. Single-band handles only. */
int bml_dev_digest(bml_dev *dev, uint64_t *digest);

/* The band's rows as a digest segment (6 words: p^cells, B[4], packed low-bit
 * map; see csrc/bml_digest.cu). bml_digest_finish() combines the segments of
 * consecutive bands (in row order) into grid_digest. Host arithmetic only. */
int bml_dev_digest_segment(bml_dev *dev, uint64_t seg[6]);
int bml_digest_finish(const uint64_t *segs, int count, uint64_t *digest);

/* The band's rows as binary-PPM pixels (3 bytes per cell, encode_ppm's body
 * without the "P6\n<n> <n>\n255\n" header; src/snapshot.cpp:21-36), written
 * to `dst` (host or device memory), rows `dst_pitch` bytes apart. */
int bml_dev_encode_ppm(bml_dev *dev, uint8_t *dst, size_t dst_pitch);

/* Vehicle counts of the band's rows (count_vehicles). */
int bml_dev_counts(bml_dev *dev, int64_t *lr, int64_t *tb);

/* Launch on an external CUDA stream (cudaStream_t passed as void*; NULL
 * restores the handle's own stream). Work already queued on the previous stream
 * is ordered before anything queued on the new one (event + stream wait). Used
 * by bench.py to time on the launching stream with CUDA events. */
int bml_dev_set_stream(bml_dev *dev, void *stream);
int bml_dev_sync(bml_dev *dev);

/* Tuning knobs (0 = keep current): temporal block depth (full steps fused per
 * launch / ghost depth of the resident kernel, 1..16, default 16) and rows per
 * warp strip of the streaming kernel (1..65536, -1 = automatic, the default;
 * rows are split evenly over rows / strip_rows strips; -ns with ns >= 2 asks
 * for exactly ns strips). */
int bml_dev_configure(bml_dev *dev, int block_steps, int strip_rows);

/* Small lattices (n % 32 == 0, n <= 1024) run the whole step loop in one
 * cluster-resident kernel (lattice kept in registers of a thread-block cluster,
 * DSMEM ghost-row exchange) unless disabled: mode 1 = auto (default), 0 = always
 * use the streaming kernel. bml_dev_path() reports the cluster size used by the
 * last bml_dev_step (0 = streaming kernel). */
int bml_dev_set_resident(bml_dev *dev, int mode);
int bml_dev_path(bml_dev *dev, int *resident_cluster);

/* Census cadence of bml_dev_step's vehicle counts on a single band: 0 = after
 * each launch's last step (default), 1 = after every step (strict: the
 * reference's per-step check, engine.cpp:219-224, at the cost of two more
 * popcounts per 32 cells per step). */
int bml_dev_set_census(bml_dev *dev, int every_step);

/* TEST HOOK (fault injection, used by tests/ only): arms a fault for the NEXT
 * bml_dev_step call — after `at_step` of its steps (0 <= at_step <= steps) the
 * cell (row, col) (band-relative row) is toggled: Empty <-> LR, TB -> Empty.
 * Up to 8 armed faults; single-band handles only. The call's launches are split
 * at the fault, so the kernels that run are the normal ones. */
int bml_dev_debug_fault(bml_dev *dev, int64_t at_step, int row, int col);

/* Streaming-kernel variant: 0 = automatic (default), 1 = narrow (32 cells per
 * lane, K <= 16 steps per launch), 2 / 3 = wide (64 cells per lane, TMA
 * bulk-copied rows, K = 14 / 12 steps per launch; n % 64 == 0 and n >= 2048
 * only, else narrow), 4 = wide with a per-lane cp.async row ring, 5 = stage-split
 * (a warp pair per item), 6 = wide in the even/odd layout (each 64-cell group held
 * as its even then its odd cells, 5 instead of 6 ALU instructions per 32 cells and
 * step; the buffer is converted in place around runs of >= 56 steps, n % 64 == 0,
 * n >= 2048, single bands and connected row bands, bare loop or metrics; anything
 * else runs the narrow kernel). Automatic (0) picks it from n >= 20480 (W >= 640).
 * Row bands: set on every band before connecting. */
int bml_dev_set_variant(bml_dev *dev, int variant);

/* The step kernel that ran the most steps of the last bml_dev_step call, and
 * how many: BML_KERNEL_NONE (no steps), _NARROW (step_block_kernel, 32 cells per
 * lane), _WIDE (step_wide_kernel, 64 cells per lane), _WIDE_EO (step_wide_kernel
 * in the even/odd layout), _SPLIT (step_split_kernel), _RESIDENT (the
 * cluster-resident kernel). For reports (bench.py's roofline names it). */
#define BML_KERNEL_NONE 0
#define BML_KERNEL_NARROW 1
#define BML_KERNEL_WIDE 2
#define BML_KERNEL_WIDE_EO 3
#define BML_KERNEL_SPLIT 4
#define BML_KERNEL_RESIDENT 5
int bml_dev_last_kernel(bml_dev *dev, int *kernel, int64_t *steps);

/* Launch geometry (row strips, work items, CTAs) of that dominant kernel's last
 * launch in the last bml_dev_step call (zeros for the resident kernel or no
 * steps); bml_dev_last_launch reports the very last launch, e.g. a run's tail. */
int bml_dev_last_kernel_launch(bml_dev *dev, int *nstrips, int *items, int *grid);

/* Geometry of the last streaming-kernel launch: row strips, work items
 * (strips x warp columns) and CTAs. */
int bml_dev_last_launch(bml_dev *dev, int *nstrips, int *items, int *grid);

/* Kernel statistics since the last reset: launches of the step kernels and
 * their summed device time (CUDA events around each launch; enable first). */
int bml_dev_enable_timing(bml_dev *dev, int enable);
int bml_dev_kernel_stats(bml_dev *dev, int64_t *launches, double *kernel_ms, int reset);

/* Geometry / introspection. */
int bml_dev_info(bml_dev *dev, int *n, int *row_begin, int *row_end, int *block_steps,
                 int *strip_rows, size_t *device_bytes);

/* ---- multi-GPU plumbing (one process per GPU, or one process driving all) ----
 * bml_dev_export() writes an opaque blob (CUDA IPC handles of the band's two
 * lattice buffers and its halo flags) of at most BML_EXPORT_BYTES bytes.
 * bml_dev_connect() maps the up-neighbour's (rows above, periodic) and
 * down-neighbour's blobs. After connect, bml_dev_step() writes halo rows
 * straight into the neighbours' buffers from inside the step kernel (NVLink
 * peer stores) and signals them with system-scope flags; no NCCL on the data
 * path. bml_dev_connect_local() does the same for handles living in this
 * process (peer access instead of IPC). */
#define BML_EXPORT_BYTES 512
int bml_dev_export(bml_dev *dev, void *blob, size_t *size);
int bml_dev_connect(bml_dev *dev, const void *up_blob, const void *down_blob);
int bml_dev_connect_local(bml_dev *dev, bml_dev *up, bml_dev *down);

/* Must be called on every band after upload/init and before the first step
 * when bands are connected: publishes boundary rows into neighbour halos. */
int bml_dev_exchange_halos(bml_dev *dev);

const char *bml_dev_last_error(void);

/* Library version / build string, e.g. "bml_dev 0.1.0 sm_100a". */
const char *bml_dev_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BML_DEV_H */
