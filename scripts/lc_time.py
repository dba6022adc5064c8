import time, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1609_01479_b200 import lb, synth
for (nx, ny, nz) in [(512, 512, 64), (128, 128, 128)]:
    n = synth.random_directors(nx, ny, nz, 0)
    with lb.LcLattice(nx, ny, nz) as L:
        L.init(n)
        L.step(3)
        for rep in range(3):
            torch.cuda.synchronize(); t = time.perf_counter(); L.step(20); t = time.perf_counter() - t
            print(nx, ny, nz, "MLUPS", nx*ny*nz*20/t/1e6, "GB/s(432)", nx*ny*nz*20*432/t/1e9, flush=True)
