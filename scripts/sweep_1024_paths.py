import ctypes, json, sys, torch
sys.path.insert(0, '.')
import paper_1804_07981_b200 as bml
n=1024; steps=4096
lat=bml.DeviceLattice(n); lat.init_random(0.38,1)
s=torch.cuda.Stream(); lat.set_stream(s.cuda_stream)
for res in (1,0):
  for k in (16,8,4):
    for strip in (-1, -16, -32, -64, -128):
      lat.set_resident(res); lat.configure(block_steps=k, strip_rows=strip)
      with torch.cuda.stream(s):
        lat.step(steps)
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(s); lat.step(steps); e1.record(s); e1.synchronize()
      print(json.dumps({"resident":res,"k":k,"strip":strip,"tcups":round(n*n*steps/(e0.elapsed_time(e1)/1e3)/1e12,3),"cluster":lat.resident_cluster}),flush=True)
      if res: break
