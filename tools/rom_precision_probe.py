"""NEXT-3 feasibility probe: a whole-domain reduced model of the
paper's 2-D cavity (101^2 cells, s = 4.95, order q, 64 excitations) stepped in
fp64, in fp32 with fp32 accumulation (what a tf32/bf16 tensor-core GEMM gives)
and in fp32 with fp64 accumulation.  python tools/rom_precision_probe.py q steps"""
import sys, math, time, numpy as np
sys.path[:0]=['/root/repo']
from oracle import yee, stability as st
from paper_1406_7042_b200.prep import reduce as rdc
from synth.scenarios import EPS0, MU0, C0, gaussian_tau
n=(101,101,1); d=(0.01,0.01,1.0)
ys=yee.assemble(2,n,d,EPS0,MU0)
De,Dm,K=ys.De,ys.Dm,ys.K.tocsr()
dtc=0.01/(C0*math.sqrt(2)); s=4.95; dt=s*dtc*0.99
rng=np.random.default_rng(7)
Ne,Nh=K.shape
nsrc=64
src=rng.choice(Ne, nsrc, replace=False)
B=np.zeros((Ne+Nh,nsrc)); B[src,np.arange(nsrc)]=1.0
q=int(sys.argv[1]) if len(sys.argv)>1 else 160
pts=rdc.expansion_points(1.1,2,3e9,dt)
t0=time.time()
V1,V2=rdc.krylov_basis(De,Dm,K,dt,B,np.arange(Ne),np.arange(Nh),q,pts)
V1=rdc.d_orthonormalise(V1,De); V2=rdc.d_orthonormalise(V2,Dm)
Kt=V1.T@(K@V2); Bt=V1.T@B[:Ne]
print("basis", V1.shape, V2.shape, time.time()-t0)
De_r=np.ones(V1.shape[1]); Dm_r=np.ones(V2.shape[1])
Kp,rep=st.enforce(De_r,Kt,Dm_r,dt)[:2] if isinstance(st.enforce(De_r,Kt,Dm_r,dt),tuple) else (st.enforce(De_r,Kt,Dm_r,dt),None)
print("sigma", np.linalg.svd(Kt,compute_uv=False)[0]*dt/2, np.linalg.svd(Kp,compute_uv=False)[0]*dt/2)
nsteps=int(sys.argv[2]) if len(sys.argv)>2 else 2000
tau=gaussian_tau(3e9); t=(np.arange(nsteps)+0.5)*dt
w=np.exp(-((t-4*tau)/tau)**2/2)
amp=rng.uniform(0.5,1.5,nsrc)
def run(dtype, acc):
    e=np.zeros((Kp.shape[0],nsrc),dtype); h=np.zeros((Kp.shape[1],nsrc),dtype)
    K_=Kp.astype(dtype); Bt_=Bt.astype(dtype); KT_=Kp.T.astype(dtype).copy()
    probes=[]
    for k in range(nsteps):
        u=(w[k]*amp)
        if acc=="f64":
            e=(e.astype(np.float64)-dt*(Kp@h.astype(np.float64))-dt*(Bt*u)).astype(dtype)
            h=(h.astype(np.float64)+dt*(Kp.T@e.astype(np.float64))).astype(dtype)
        else:
            e=(e-(np.float32(dt)*(K_@h))-(np.float32(dt)*(Bt_*u.astype(dtype)))).astype(dtype)
            h=(h+np.float32(dt)*(KT_@e)).astype(dtype)
        probes.append((V1[src[:4]]@e.astype(np.float64)).diagonal().copy() if False else float(np.linalg.norm(e)))
    return e.astype(np.float64),h.astype(np.float64),np.array(probes)
e0,h0,p0=run(np.float64,"f64")
for dtype,acc in ((np.float32,"f32"),(np.float32,"f64")):
    e,h,p=run(dtype,acc)
    print(acc, "e", np.linalg.norm(e-e0)/np.linalg.norm(e0), "h", np.linalg.norm(h-h0)/np.linalg.norm(h0))
