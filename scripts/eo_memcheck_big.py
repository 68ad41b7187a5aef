"""compute-sanitizer target: the pitch-specialised even/odd kernel (the N=32768
instantiation, immediate row offsets, zero pad rows past the band end) for one 60-step
run on a device-drawn lattice; prints the digest and vehicle counts for the log
(bit-exactness of that kernel is covered by tests/test_gpu_eo.py's goldens)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

for n in (32768,):
    lat = bml.DeviceLattice(n)
    lat.init_random(0.35, 1)
    lat.step(60)
    print(n, hex(lat.digest()), lat.counts(), flush=True)
