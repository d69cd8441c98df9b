import time, numpy as np, sys, os
sys_path_fix = __import__("sys").path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1905_12799_b200 import _lib
rng=np.random.default_rng(0)
res=[]
for m in (64,200,500):
    X=rng.integers(0,10,size=(m,4)).astype(np.float64); y=rng.random(m)
    C=_lib.C; per=(1<<5)-1; cap=50*per
    feat=np.zeros(cap,np.int32); thr=np.zeros(cap); left=np.zeros(cap,np.int32); right=np.zeros(cap,np.int32); val=np.zeros(cap); offs=np.zeros(51,np.int32); base=C.c_double()
    args=(_lib.as_ptr(X,C.c_double),_lib.as_ptr(y,C.c_double),m,4,50,4,0.3,_lib.as_ptr(feat,C.c_int32),_lib.as_ptr(thr,C.c_double),_lib.as_ptr(left,C.c_int32),_lib.as_ptr(right,C.c_int32),_lib.as_ptr(val,C.c_double),cap,_lib.as_ptr(offs,C.c_int32),C.byref(base))
    best=1e9
    for r in range(7):
        t=time.perf_counter()
        for _ in range(10): _lib.call("kt_fit_trees",*args)
        best=min(best,(time.perf_counter()-t)/10)
    res.append(f"m={m}: {best*1e6:.0f} us")
print(os.environ.get("KT_LIB_PATH","in-tree"), *res)
