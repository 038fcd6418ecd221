#!/usr/bin/env python3
"""Register-reuse feasibility of the cubic SL gather: for voxel pairs /
quads of one thread along axis 0, how often their other-axis stencil bases coincide
per lane and for all 32 lanes of a warp, on the analytic bench rotation (half and
full amplitude) and a generic smooth 3D field.  usage: tools/reuse_sim.py rot|rotfull|gen"""
import numpy as np, sys
n = 256
rng = np.random.default_rng(0)
h = 2*np.pi/n
def coords(j): return (n//2 - (j+1.0))*h
def field(case, i, j, k):
    x0, x1, x2 = coords(i), coords(j), coords(k)
    if case.startswith("rot"):
        amp = 0.35 if case == "rot" else 0.7
        mod = 1 + 0.3*np.cos(x2)
        return -amp*np.cos(x0)*np.sin(x1)*mod, amp*np.sin(x0)*np.cos(x1)*mod, 0*x0
    # generic smooth 3D field: sum of a few random low modes, max |v| ~ amp
    amp = 0.5
    r = np.random.default_rng(5)
    v = [0*x0, 0*x0, 0*x0]
    for c in range(3):
        for m in range(4):
            kk = r.integers(-2, 3, 3); ph = r.uniform(0, 6.28)
            v[c] = v[c] + amp/4*np.sin(kk[0]*x0 + kk[1]*x1 + kk[2]*x2 + ph)
    return v
case = sys.argv[1]
NW = 40000
i0 = rng.integers(0, n//4, NW)*4; j0 = rng.integers(0, n, NW); k0 = rng.integers(0, n//32, NW)*32
lane = np.arange(32)
s = 0.25/h
def bases(i, j, k):
    v = field(case, i % n, j % n, k % n)
    return [np.floor(c*s).astype(int) for c in v]   # floor(d) per axis (index shift cancels in deltas)
B = [bases(i0[:, None] + u, j0[:, None] + 0*lane, k0[:, None] + lane) for u in range(4)]
for pr in [(0, 1), (2, 3)]:
    a, b = B[pr[0]], B[pr[1]]
    d0 = b[0] - a[0]; d1 = b[1] - a[1]; d2 = b[2] - a[2]
    static = (d0 == 0) & (d1 == 0) & (d2 == 0)   # delta of floor(d): plane step 1, same rows, same cols
    print(f"{case} pair{pr}: lane static {static.mean():.3f}  warp all-static {static.all(1).mean():.3f}  "
          f"warp |dfloor|<=1 all axes {((abs(d0)<=1)&(abs(d1)<=1)&(abs(d2)<=1)).all(1).mean():.3f} "
          f"warp d1,d2==0 {((d1==0)&(d2==0)).all(1).mean():.3f}")
# quad: all 4 voxels share rows/cols and step 1 planes
st = np.ones((NW, 32), bool)
for u in range(1, 4):
    for ax in range(3):
        st &= (B[u][ax] == B[0][ax])
print(f"{case} quad: lane static {st.mean():.3f}  warp static {st.all(1).mean():.3f}")
