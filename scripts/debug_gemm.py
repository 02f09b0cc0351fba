import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_gpu_kernels import _gemm
from paper_1802_07170_b200 import _lib
for shape in [(128,128,40),(128,128,64),(64,128,64),(128,96,64),(16,128,128),(16,64,128),(128,128,32),(128,64,128),(128,32,128)]:
    for (am,bm) in [(0,1),(0,0),(1,1)]:
        for bn in [64,128]:
            M,N,K=shape
            C,ref=_gemm(_lib.MODE_BF16,M,N,K,am,bm,bn)
            err=((C-ref).abs().max()/ref.abs().max()).item()
            print(shape,am,bm,bn,"%.2e"%err, flush=True)
from oracle import minmt_oracle as O
from tests.gpu_helpers import engine_step, oracle_step, scaled_params
for case in [(1000,128,128,1,16,20,20),(1000,128,128,2,16,20,20),(256,128,128,1,16,9,8),(256,64,64,1,16,9,8)]:
    V,E,H,L,B,S,T=case
    d=O.Dims(V,E,H,L,0.2)
    params=scaled_params(d,3,0.1); batch=O.synthetic_batch(V,S,T,B,seed=4,ragged=True)
    ol,_,og,_,_=oracle_step(d,params,batch,0.1,1.0,5.0,21,update=False)
    for mode in ["fp32","bf16"]:
        loss,_,g,_,_=engine_step(d,params,batch,0.1,1.0,5.0,21,mode,update=False)
        errs={n:O.norm_rel_err(g[n],og[n]) for n in g}
        bad={n:"%.1e"%e for n,e in errs.items() if e>2e-2}
        print(case,mode,"loss",loss,ol,"worst","%.2e"%max(errs.values()),bad, flush=True)
