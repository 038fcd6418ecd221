"""Event-timed reg preconditioner apply at 256^3 (debug helper)."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2401_17493_b200 as F
n=256
m0,m1,vt=F.synth_case("rotation",n,seed=1,d=3)
st=F.KktState(m0,m1,F.RegConfig(alpha=1e-2),v_init=F.VectorField._wrap(m0.grid,0.5*vt.data),transport_dtype=np.float32)
r=F.VectorField._wrap(m0.grid, torch.randn((3,n,n,n),dtype=torch.float64,device="cuda"))
pk=F.PrecondKind("reg")
for _ in range(3): st.apply_precond(r,pk,0.1)
torch.cuda.synchronize()
a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): st.apply_precond(r,pk,0.1)
b.record(); torch.cuda.synchronize(); print("precond ms", a.elapsed_time(b)/10)
