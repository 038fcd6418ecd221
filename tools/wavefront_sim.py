#!/usr/bin/env python3
"""Shared-memory wavefronts per voxel of the cubic gather: the shipped LDS.32 scheme vs
x-pairs reading 8-column LDS.128 windows (bank groups of 16-B blocks, duplicate
blocks merged as measured in profiles/r02_lds_microbench.txt).  usage: tools/wavefront_sim.py rot|swirl"""
n = 256
import numpy as np, sys
n = 256
rng = np.random.default_rng(0)
case = sys.argv[1] if len(sys.argv) > 1 else "rot"
amp = {"rot": 0.35, "rotfull": 0.7, "swirl": 0.6}[case]
h = 2*np.pi/n
def coords(j): return (n//2 - (j+1.0))*h
NW = 20000
# warp origins: x-run of 32 lanes (Z scheme) ; 64 voxels along x for X scheme
i0 = rng.integers(0, n, NW); j0 = rng.integers(0, n, NW); k0 = rng.integers(0, n//64, NW)*64
def disp(i, j, k):
    x0, x1, x2 = coords(i), coords(j), coords(k)
    mod = 1 + 0.3*np.cos(x2)
    p0, p1 = (0.0, 0.0) if case != "swirl" else (0.7, -1.3)
    v0 = -amp*np.cos(x0-p0)*np.sin(x1-p1)*mod
    v1 = amp*np.sin(x0-p0)*np.cos(x1-p1)*mod
    if case == "swirl":
        v0 += -0.5*amp*0.5*np.cos(2*(x0-0.4))*np.sin(x1+0.9)
        v1 += 0.5*amp*np.sin(2*(x0-0.4))*np.cos(x1+0.9)
    s = 0.25/h  # dt / h in index units (sign irrelevant for stats)
    return v0*s, v1*s, 0*v0
def bases(i, j, k):
    d0, d1, d2 = disp(i, j, k)
    return (i + np.floor(d0)).astype(np.int64), (j + np.floor(d1)).astype(np.int64), (k + np.floor(d2)).astype(np.int64)
def wf_count(addr_words, width):
    # addr_words: (NW, 32) word address of each lane's access (aligned to width words)
    # wavefronts = max over bank-groups of distinct addresses in the group
    unit = addr_words // width
    G = 32 // width
    grp = unit % G
    tot = 0
    for g in range(G):
        m = grp == g
        a = np.where(m, unit, -1)
        a = np.sort(a, axis=1)
        distinct = ((a[:, 1:] != a[:, :-1]) & (a[:, 1:] >= 0)).sum(1) + (a[:, 0] >= 0)
        tot = np.maximum(tot, distinct) if g else distinct
    return tot
P, R = 1024, 64   # plane / row pitch in words (box 12x16x64)
# ---------- Z scheme (current): lane l = x k0+l (first 32 of the 64), 64 LDS.32 per voxel
lane = np.arange(32)
I = i0[:, None] + 0*lane; J = j0[:, None] + 0*lane; K = k0[:, None] + lane
b0, b1, b2 = bases(I % n, J % n, K % n)
wz = 0
for a in range(4):
    for b in range(4):
        for t in range(4):
            wz = wz + wf_count((b0 + a)*P + (b1 + b)*R + (b2 + t) % 64 + 64*0, 1)
print(f"Z: wavefronts per voxel {wz.mean()/32:.3f}  (64 LDS.32 / voxel)")
# ---------- X scheme: lane l = voxels (k0+2l, k0+2l+1)
KA = k0[:, None] + 2*lane; KB = KA + 1
a0, a1, a2 = bases(I % n, J % n, KA % n)
c0, c1, c2 = bases(I % n, J % n, KB % n)
dz = c0 - a0; dy = c1 - a1; dx = c2 - a2
print("x-pair mismatch: dz!=0 %.3f  dy!=0 %.3f  dx dist" % ((dz != 0).mean(), (dy != 0).mean()), np.unique(dx, return_counts=True))
lo0 = np.minimum(a0, c0); lo1 = np.minimum(a1, c1)
NPl = 4 + np.abs(dz).max(1); NRw = 4 + np.abs(dy).max(1)   # warp-uniform union window
cmin = np.minimum(a2, c2) - 1; cmax = np.maximum(a2, c2) + 2
W0 = (cmin // 4) * 4
nblk = (cmax - W0) // 4 + 1       # 2 or 3
NB = nblk.max(1)
print("warps needing 5 planes %.3f, 5+ rows %.3f, 3 blocks %.3f" % ((NPl > 4).mean(), (NRw > 4).mean(), (NB > 2).mean()))
wx = 0; instr = 0
for a in range(5):
    for b in range(6):
        for q in range(3):
            act = (a < NPl) & (b < NRw) & (q < NB)
            w = wf_count((lo0 - 1 + a)*P + (lo1 - 1 + b)*R + (W0 + 4*q) % 64 + 0, 4)
            wx = wx + np.where(act, w, 0)
            instr = instr + act
print(f"X: wavefronts per voxel {wx.mean()/64:.3f}  LDS.128 per voxel {instr.mean()/2:.1f}  rows per plane {NRw.mean():.2f} planes {NPl.mean():.2f} blocks {NB.mean():.2f}")
