"""compute-sanitizer target: the pitch-specialised even/odd kernels (N=32768 and 65536
instantiations are only used at those sizes) for one 60-step run each, digest checked
against the unmodified reference's golden where one exists at 60 steps (none: the
digest is printed for the log), plus the N=32768 10000-step golden at the end."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

for n in (32768,):
    lat = bml.DeviceLattice(n)
    lat.init_random(0.35, 1)
    lat.step(60)
    print(n, hex(lat.digest()), lat.counts(), flush=True)
