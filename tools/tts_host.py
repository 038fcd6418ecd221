import cProfile, pstats, sys, os, time, gc, io
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2401_17493_b200 as F
m0, m1, v = F.synth_case("rotation", 256, seed=1, d=3)
reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
def run():
    torch.cuda.synchronize(); t0 = time.perf_counter()
    vs, r = F.register(m0, m1, reg=reg, precond=F.PrecondKind("reg"), transport_dtype=np.float32)
    torch.cuda.synchronize(); return time.perf_counter() - t0
print("plain", [round(run(), 3) for _ in range(6)])
gc.disable()
print("gc off", [round(run(), 3) for _ in range(6)])
gc.enable()
pr = cProfile.Profile()
walls = []
for _ in range(4):
    pr.enable(); walls.append(run()); pr.disable()
print("profiled", walls)
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue()[:6000])
