import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import fdirw_inputs as fi
import paper_2408_11376_b200 as fd
shape=(9,10,11)
m=fi.porous_particle(shape,4,pore_r=(1.0,1.5),n_pores=3,seed=4)
for R in (5,8):
    p=fd.Params(nx=11,ny=10,nz=9,dh=1.0,D_fast=1.0,D_slow=1e-3,dt=3.0,radius=R,n_fd=0,weights="bf16",flags=0,v_far=0.0)
    with fd.build_kernels(p,m) as ctx: pass
print("ok")
