import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1905_12799_b200 as kt
from paper_1905_12799_b200 import _lib
eng = kt.engine(0)
def run(ta, tb, A, B):
    M, K = A.shape; N = B.shape[1]
    Ag = np.ascontiguousarray(A.T if ta else A).astype(np.float32); Bg = np.ascontiguousarray(B.T if tb else B).astype(np.float32)
    with eng.scope():
        dA, dB = torch.from_numpy(Ag).cuda(), torch.from_numpy(Bg).cuda()
        dC = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        _lib.call("kt_gemm_f32", eng.handle, ta, tb, M, N, K, _lib.ptr(dA), Ag.shape[1], _lib.ptr(dB), Bg.shape[1], _lib.ptr(dC), N)
        return dC.cpu().numpy()
M, N, K = 128, 32, 32
rng = np.random.default_rng(0)
for ta in (0, 1):
    for tb in (0, 1):
        A = rng.standard_normal((M, K)); B = rng.standard_normal((K, N))
        C = run(ta, tb, A, B); err = np.abs(C - A @ B).max()
        print(f"ta={ta} tb={tb} err={err:.2e}")
        if err > 1e-3:
            # probe: A = e_{m,k} one-hot, B = code matrix: B[k][n] = 1000*k + n  -> C[m][n] = B[k][n]
            for (m, k) in [(0, 0), (1, 0), (0, 1), (8, 0), (0, 4), (0, 8), (5, 3), (9, 6)]:
                A1 = np.zeros((M, K)); A1[m, k] = 1.0
                Bc = np.array([[1000.0 * kk + n for n in range(N)] for kk in range(K)])
                C1 = run(ta, tb, A1, Bc)
                nz = np.argwhere(np.abs(C1) > 0.5)
                rows = sorted(set(nz[:, 0].tolist()))
                vals = C1[rows[0]][:4] if rows else None
                print(f"   A[{m},{k}]=1 -> nonzero rows {rows[:6]} first vals {vals}")
