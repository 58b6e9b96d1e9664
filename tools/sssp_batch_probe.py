"""Batch-size probe of the device SSSP cost build (k_sssp.cu): the one-call
build of the office and bridge scenes with DPSO_SSSP_BATCH concurrent
sources ("0" = the built-in choice), median of 7 (host-timed: each call
syncs), and that every batch size gives the same matrix.

    python tools/sssp_batch_probe.py > profiles/r02/sssp_batch_probe.jsonl
"""
import os, sys, time, json, ctypes
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tools')
import numpy as np, torch, scenes
from paper_1706_04399_b200 import _lib
from paper_1706_04399_b200.graph import _grid_args
lib=_lib.load()
for name in ("office","bridge"):
    occ,vox,w=scenes.scene(name); o,v,wt=_grid_args(occ,vox,w); n=len(v)
    docc=torch.from_numpy(o.ravel()).cuda(); ld=(n+7)//8*8
    cost=torch.zeros((n,ld),dtype=torch.float64,device='cuda'); virt=torch.zeros((n,n),dtype=torch.uint8,device='cuda')
    ref=None
    for _ in range(3):
        vc=ctypes.c_double(); _lib.check(lib.dpso_build_cost(docc.data_ptr(),*o.shape,wt.ctypes.data_as(ctypes.c_void_p),v.ctypes.data_as(ctypes.c_void_p),n,cost.data_ptr(),ld,virt.data_ptr(),ctypes.byref(vc),None))
    for B in ("0","1024","256","128","96","64","32"):
        if B=="0": os.environ.pop("DPSO_SSSP_BATCH",None)
        else: os.environ["DPSO_SSSP_BATCH"]=B
        ts=[]
        for r in range(7):
            vc=ctypes.c_double(); torch.cuda.synchronize(); t=time.perf_counter()
            _lib.check(lib.dpso_build_cost(docc.data_ptr(),*o.shape,wt.ctypes.data_as(ctypes.c_void_p),v.ctypes.data_as(ctypes.c_void_p),n,cost.data_ptr(),ld,virt.data_ptr(),ctypes.byref(vc),None))
            torch.cuda.synchronize(); ts.append(time.perf_counter()-t)
        c=cost.cpu().numpy()
        if ref is None: ref=c
        print(json.dumps({"scene":name,"B":B,"median_ms":round(float(np.median(ts))*1e3,1),"min_ms":round(min(ts)*1e3,1),"same":bool(np.array_equal(c,ref))}),flush=True)
