import sys, time, torch
sys.path.insert(0, '.')
from paper_1609_01479_b200 import lb, synth
for (n, K) in [(64, 1000), (128, 200), (512, 100)]:
    nz = 64 if n == 512 else n
    L = lb.Lattice(n, n, nz)
    L.init_equilibrium(synth.spinodal_phi(n, n, nz, 0))
    st = torch.cuda.ExternalStream(lb.lb_stream(L.h))
    L.step(5)
    for prof in (False, True, False, True):
        lb.lb_profile_enable(L.h, prof)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(st); L.step(K); e1.record(st); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        print(n, nz, "prof" if prof else "plain", f"{ms*1e3:.1f} us/step", f"{n*n*nz/ms/1e3:.0f} MLUPS", flush=True)
    L.close()
