"""tcgen05 3xTF32 GEMM (kt_gemm_f32) against a float64 reference: fp32-level accuracy on every layout."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_12799_b200 as kt  # noqa: E402
from paper_1905_12799_b200 import _lib  # noqa: E402


@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("shape", [(128, 128, 128), (1000, 25, 128), (77, 64, 8), (4096, 128, 130), (130, 48, 3000),
                                   (128, 16, 32), (300, 200, 64)])
def test_gemm_layouts(ta, tb, shape):
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    Ag = np.ascontiguousarray(A.T if ta else A)
    Bg = np.ascontiguousarray(B.T if tb else B)
    eng = kt.engine(0)
    with eng.scope():
        dA, dB = torch.from_numpy(Ag).cuda(), torch.from_numpy(Bg).cuda()
        dC = torch.empty((M, N), dtype=torch.float32, device="cuda")
        lda, ldb = Ag.shape[1], Bg.shape[1]
        _lib.call("kt_gemm_f32", eng.handle, ta, tb, M, N, K, _lib.ptr(dA), lda, _lib.ptr(dB), ldb, _lib.ptr(dC), N)
        C = dC.cpu().numpy()
    want = A.astype(np.float64) @ B.astype(np.float64)
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
    err = np.abs(C - want) / np.maximum(scale, 1e-30)
    # fp32-accurate products (plain TF32 would be ~1e-3); fp32 accumulation error grows ~sqrt(K)
    assert err.max() < 1e-6 + 1e-7 * np.sqrt(K), err.max()
