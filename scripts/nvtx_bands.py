"""Two row bands of an N=8192 torus on one GPU (in-kernel ghost exchange), a few
launches each, for an NVTX-attributed ncu launch list: every kernel shows the
C-ABI range ("bml" domain) it was launched from (bml_dev_init_random,
bml_dev_exchange_halos, bml_dev_step, bml_dev_digest_segment)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

lat = bml.DeviceLattice(8192, 2)
lat.configure(block_steps=16, strip_rows=0)
lat.init_random(0.35, 1)
lat.step(48)
print(hex(lat.digest()))
