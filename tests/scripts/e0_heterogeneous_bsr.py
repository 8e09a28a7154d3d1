"""Experiment behind reading A24: inexact BSR V(1,1) with the lognormal K field of
config 4 (sigma = 2) on 32^2, 4 levels, oracle only.  The smoother alone converges (rho 0.96-0.98)
but every cycle variant diverges: coarse K^{-1} by arithmetic mean (A11), coarse K by arithmetic
mean, and Galerkin coarse M_w = P_w^T M_w P_w."""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
import mg_inputs
from oracle.cycle import Hierarchy
import oracle.cycle as oc
n=32; L=4
Kf=mg_inputs.lognormal_K(n,3)
def rho_cycle(H, opts, cycles=30):
    r,rs=H.measure_rho(opts, seed=0, min_cycles=cycles, max_cycles=cycles); return float(np.mean(rs[-4:]))
def rho_smoother(H, opts, sweeps=60):
    rng=np.random.default_rng(0); N=H.ops[0].A.shape[0]; x=rng.uniform(-1,1,N); b=np.zeros(N)
    prev=np.linalg.norm(H.ops[0].A@x); rs=[]
    for _ in range(sweeps):
        x=H.smooth(0,x,b,opts); r=np.linalg.norm(H.ops[0].A@x); rs.append(r/prev); prev=r
    return float(np.mean(rs[-5:]))
orig=oc.coarsen_Kinv
def harmonic(fine, coarse, Kinv_f):
    # coarse K = mean of the children's K  (K^{-1} = 1 / mean(1/K^{-1}))
    Kc = orig(fine, coarse, 1.0/Kinv_f)
    return 1.0/Kc
for name,fn in (('arith_Kinv',orig),('arith_K',harmonic)):
    oc.coarsen_Kinv=fn
    H=Hierarchy(n,L,1.0,1.0,1.0,1.0,1.0,1.0,Kinv_field=1.0/Kf,relax='bsr')
    for (omJ,om) in ((0.7,0.3),(1.0,0.5),(0.7,0.6),(1.0,0.8)):
        o=dict(nu1=1,nu2=1,omega=om,omega_J=omJ,jacobi_sweeps=3)
        print(name,(omJ,om),'cycle rho',round(rho_cycle(H,o),3),'smoother rho',round(rho_smoother(H,o),4), flush=True)
oc.coarsen_Kinv=orig
print('--- Galerkin M_w on coarse levels')
import scipy.sparse as sp
from oracle.relax import BSR
H=Hierarchy(n,L,1.0,1.0,1.0,1.0,1.0,1.0,Kinv_field=1.0/Kf,relax='bsr')
for l in range(1,L):
    opf, opc, T = H.ops[l-1], H.ops[l], H.transfers[l-1]
    Pw = T.mats['P_w'].tocsr()
    mf, mc = H.meshes[l-1], H.meshes[l]
    Mwf = opf.full['Mw'] if l==1 else H._gal_full
    MwG = (Pw.T @ Mwf @ Pw).tocsr()
    H._gal_full = MwG
    act=mc.act_idx
    A_full = opc.A_full - opc.tau*opc.full['Mw'] + opc.tau*MwG
    opc.A_full=A_full.tocsr(); opc.A=A_full.tocsr()[act][:,act].tocsr()
    kind=mc.slot_kind(act); sw=act[(kind>=5)&(kind<=7)]
    opc.Mw=MwG[sw][:,sw].tocsr()
    if l < L-1: H.smoothers[l]=BSR(opc)
H.coarse=oc.CoarseSolver(H.ops[-1])
for (omJ,om) in ((0.7,0.3),(1.0,0.5),(0.7,0.6),(1.0,0.8)):
    o=dict(nu1=1,nu2=1,omega=om,omega_J=omJ,jacobi_sweeps=3)
    print('galerkin Mw',(omJ,om),'cycle rho',round(rho_cycle(H,o),3), flush=True)
