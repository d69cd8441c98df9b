import sys, numpy as np, torch
sys.path.insert(0, '.')
exec(open('tools/gemm_debug.py').read().split('M, N, K = 128')[0])
for (M,N,K) in [(130,48,3000),(128,48,3000),(130,48,64),(256,48,3000),(130,48,1000)]:
    for ta in (0,1):
        rng=np.random.default_rng(1); A=rng.standard_normal((M,K)); B=rng.standard_normal((K,N))
        C=run(ta,0,A,B); W=A@B; S=np.abs(A)@np.abs(B); e=np.abs(C-W)/S
        bad=np.argwhere(e>2e-6)
        print(M,N,K,'ta',ta,'max',e.max(), 'bad rows', sorted(set(bad[:,0].tolist()))[:10], len(bad))
