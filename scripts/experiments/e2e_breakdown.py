"""Per-call host time of the e2e leg (upload / step / download) through the C-ABI.
python scripts/experiments/e2e_breakdown.py [n steps]"""
import ctypes
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
lib = ctypes.CDLL(os.environ.get("BML_LIB", os.path.join(ROOT, "paper_1804_07981_b200", "libbml_dev.so")))
vp = ctypes.c_void_p
lib.bml_dev_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
lib.bml_dev_upload.argtypes = [vp, vp, ctypes.c_size_t]
lib.bml_dev_download.argtypes = [vp, vp, ctypes.c_size_t]
lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
h = vp()
assert lib.bml_dev_create(n, 0, ctypes.byref(h)) == 0
host_in = torch.randint(0, 3, (n * n,), dtype=torch.uint8).pin_memory()
host_out = torch.empty(n * n, dtype=torch.uint8).pin_memory()
res = {"upload": [], "step": [], "download": [], "step0": []}
for i in range(25):
    t0 = time.perf_counter()
    assert lib.bml_dev_upload(h, vp(host_in.data_ptr()), n) == 0
    t1 = time.perf_counter()
    assert lib.bml_dev_step(h, steps, None, None, None, None) == 0
    t2 = time.perf_counter()
    assert lib.bml_dev_download(h, vp(host_out.data_ptr()), n) == 0
    t3 = time.perf_counter()
    assert lib.bml_dev_step(h, 0, None, None, None, None) == 0
    t4 = time.perf_counter()
    if i >= 5:
        res["upload"].append(t1 - t0)
        res["step"].append(t2 - t1)
        res["download"].append(t3 - t2)
        res["step0"].append(t4 - t3)
print({k: round(statistics.median(v) * 1e6, 1) for k, v in res.items()}, "us, n =", n, "steps =", steps)
