"""Row-band decomposition across processes (one process per GPU).

The reference parallelises only with std::thread row bands inside one process
(/root/reference/proj/src/engine.cpp:124-142, contiguous bands of ceil(n/T) rows).
Here each rank owns one band of ceil(n/world) rows on its own GPU. Bootstrap uses
torch.distributed (any backend) to all-gather the bands' CUDA-IPC export blobs;
after that the data path has no collective at all: the step kernel itself stores
the band's first/last 16 rows into the neighbours' ghost rows over NVLink and
raises a system-scope flag (include/bml_dev.h, bml_dev_connect).

Everything above the C-ABI is plain Python so the host logic (partitioning,
neighbour selection, blob exchange) is testable on CPU with the gloo backend.
"""
import ctypes
import os

from . import LIB_DEV

EXPORT_BYTES = 512  # BML_EXPORT_BYTES in include/bml_dev.h
MIN_BAND_ROWS = 16


def band_rows(n, world, rank):
    """Rows [begin, end) of `rank`'s band: parallel_rows_phase's split (engine.cpp:131-137)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    band = (n + world - 1) // world
    begin = min(n, rank * band)
    end = min(n, begin + band)
    return begin, end


def check_partition(n, world):
    """Every band must hold >= 16 rows (the ghost depth); raises ValueError otherwise."""
    for r in range(world):
        b, e = band_rows(n, world, r)
        if e - b < MIN_BAND_ROWS:
            raise ValueError(f"n={n} over {world} ranks leaves rank {r} with {e - b} rows (< 16)")


def neighbour_ranks(rank, world):
    """(up, down): the bands holding the rows just above / below, periodic (torus)."""
    return (rank - 1) % world, (rank + 1) % world


def exchange_blobs(blob, group=None):
    """All-gather every rank's export blob (bytes) through torch.distributed."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, bytes(blob), group=group)
    return out


def weak_scaled_n(n1, world):
    """Square lattice with ~world x the cells of an n1 x n1 lattice, side a multiple of 32."""
    import math

    return max(32, int(round(n1 * math.sqrt(world) / 32.0)) * 32)


class _Abi:
    def __init__(self):
        lib = ctypes.CDLL(LIB_DEV)
        vp = ctypes.c_void_p
        lib.bml_dev_create_band.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(vp)]
        lib.bml_dev_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
        lib.bml_dev_destroy.argtypes = [vp]
        lib.bml_dev_upload.argtypes = [vp, vp, ctypes.c_size_t]
        lib.bml_dev_download.argtypes = [vp, vp, ctypes.c_size_t]
        lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
        lib.bml_dev_last_kernel.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)]
        lib.bml_dev_counts.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        lib.bml_dev_export.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_size_t)]
        lib.bml_dev_connect.argtypes = [vp, vp, vp]
        lib.bml_dev_exchange_halos.argtypes = [vp]
        lib.bml_dev_init_random.argtypes = [vp, ctypes.c_double, ctypes.c_uint64]
        lib.bml_dev_digest_segment.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
        lib.bml_digest_finish.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_uint64)]
        lib.bml_dev_sync.argtypes = [vp]
        lib.bml_dev_set_stream.argtypes = [vp, vp]
        lib.bml_dev_configure.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        lib.bml_dev_enable_timing.argtypes = [vp, ctypes.c_int]
        lib.bml_dev_kernel_stats.argtypes = [vp, ctypes.POINTER(ctypes.c_int64),
                                             ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        lib.bml_dev_last_error.restype = ctypes.c_char_p
        self.lib = lib

    def check(self, rc, what):
        if rc != 0:
            msg = self.lib.bml_dev_last_error().decode()
            if rc == 1:
                raise ValueError(f"{what}: {msg}")
            raise RuntimeError(f"{what}: rc={rc}: {msg}")


class BandLattice:
    """This rank's band of an n x n torus, connected to its neighbours' processes."""

    def __init__(self, n, rank, world, device, group=None, block_steps=16, strip_rows=0):
        check_partition(n, world)
        self.abi = _Abi()
        self.n, self.rank, self.world = n, rank, world
        self.begin, self.end = band_rows(n, world, rank)
        self.h = ctypes.c_void_p()
        self.abi.check(self.abi.lib.bml_dev_create_band(n, self.begin, self.end, device,
                                                        ctypes.byref(self.h)), "create_band")
        self.abi.check(self.abi.lib.bml_dev_configure(self.h, block_steps, strip_rows), "configure")
        if world > 1:
            buf = ctypes.create_string_buffer(EXPORT_BYTES)
            size = ctypes.c_size_t(EXPORT_BYTES)
            self.abi.check(self.abi.lib.bml_dev_export(self.h, buf, ctypes.byref(size)), "export")
            blobs = exchange_blobs(buf.raw[: size.value], group)
            up, down = neighbour_ranks(rank, world)
            ub = ctypes.create_string_buffer(blobs[up], len(blobs[up]))
            db = ctypes.create_string_buffer(blobs[down], len(blobs[down]))
            self.abi.check(self.abi.lib.bml_dev_connect(self.h, ub, db), "connect")

    @property
    def rows(self):
        return self.end - self.begin

    def upload_rows(self, data, pitch=None):
        """`data`: bytes-like or pointer of this band's rows (row `begin` first)."""
        pitch = pitch or self.n
        if isinstance(data, int):
            ptr = data
        else:
            buf = (ctypes.c_char * len(data)).from_buffer_copy(data)
            self._keep = buf
            ptr = ctypes.addressof(buf)
        self.abi.check(self.abi.lib.bml_dev_upload(self.h, ctypes.c_void_p(ptr), pitch), "upload")

    def init_random(self, rho, seed):
        """This band's rows of the reference init_grid({n, rho, seed}) lattice,
        generated on the device (bml_dev_init_random); call exchange_halos() next."""
        self.abi.check(self.abi.lib.bml_dev_init_random(self.h, rho, seed), "init_random")

    def exchange_halos(self):
        self.abi.check(self.abi.lib.bml_dev_exchange_halos(self.h), "exchange_halos")

    def step(self, steps):
        self.abi.check(self.abi.lib.bml_dev_step(self.h, steps, None, None, None, None), "step")

    def download_rows(self):
        out = ctypes.create_string_buffer(self.rows * self.n)
        self.abi.check(self.abi.lib.bml_dev_download(self.h, out, self.n), "download")
        return out.raw

    def counts(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self.abi.check(self.abi.lib.bml_dev_counts(self.h, ctypes.byref(a), ctypes.byref(b)), "counts")
        return a.value, b.value

    def digest_segment(self):
        """This band's grid_digest segment (6 words), computed on the device."""
        seg = (ctypes.c_uint64 * 6)()
        self.abi.check(self.abi.lib.bml_dev_digest_segment(self.h, seg), "digest_segment")
        return list(seg)

    def set_stream(self, stream_ptr):
        self.abi.check(self.abi.lib.bml_dev_set_stream(self.h, ctypes.c_void_p(stream_ptr)), "set_stream")

    def synchronize(self):
        self.abi.check(self.abi.lib.bml_dev_sync(self.h), "sync")

    def enable_timing(self, on=True):
        self.abi.check(self.abi.lib.bml_dev_enable_timing(self.h, 1 if on else 0), "timing")

    def last_kernel(self):
        """BML_KERNEL_* of the step kernel that ran most of the last step() call."""
        k, st = ctypes.c_int(), ctypes.c_int64()
        self.abi.check(self.abi.lib.bml_dev_last_kernel(self.h, ctypes.byref(k), ctypes.byref(st)), "last_kernel")
        return k.value

    def kernel_stats(self, reset=False):
        n = ctypes.c_int64()
        ms = ctypes.c_double()
        self.abi.check(self.abi.lib.bml_dev_kernel_stats(self.h, ctypes.byref(n), ctypes.byref(ms),
                                                         1 if reset else 0), "kernel_stats")
        return n.value, ms.value

    def close(self):
        if self.h:
            self.abi.lib.bml_dev_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def combine_digest(segments):
    """grid_digest of the whole torus from every band's segment, in band (row) order."""
    lib = _Abi().lib
    flat = (ctypes.c_uint64 * (6 * len(segments)))(*[w for seg in segments for w in seg])
    out = ctypes.c_uint64()
    rc = lib.bml_digest_finish(flat, len(segments), ctypes.byref(out))
    if rc != 0:
        raise RuntimeError("bml_digest_finish failed")
    return out.value


def init_from_env():
    """torchrun-style env -> (rank, world, local_rank)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))
