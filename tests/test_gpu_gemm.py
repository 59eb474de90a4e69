"""tcgen05 TF32 GEMM vs a plain torch fp64 reference: all operand majors, tile
widths, split-K with ragged M, and CTA pairs (cta_group::2, 256-row tiles)."""

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def run(M, N, K, a_trans, b_trans, splits=1, bn=128, pair=1):
    from paper_2604_07239_b200 import _native
    lib = _native.lib()
    g = torch.Generator(device="cuda").manual_seed(M * 131 + N * 7 + K)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(K, N, device="cuda", generator=g)
    As = A.t().contiguous() if a_trans else A.contiguous()       # [K][M] or [M][K]
    Bs = B.t().contiguous() if b_trans else B.contiguous()       # [N][K] or [K][N]
    ldc = (N + 3) // 4 * 4
    C = torch.full((splits, M, ldc), float("nan"), device="cuda")
    st = lib.fade_debug_gemm(As.data_ptr(), As.shape[1], a_trans, Bs.data_ptr(), Bs.shape[1],
                             b_trans, C.data_ptr(), ldc, M, N, K, splits, bn, pair, None)
    assert st == 0, _native.last_error()
    torch.cuda.synchronize()
    ref = (A.double() @ B.double())
    kt = (K + 31) // 32
    per = -(-kt // max(1, min(splits, kt)))
    used = -(-kt // per)
    got = C[:used, :, :N].double().sum(0)
    return (got - ref).abs().max().item() / max(1e-9, ref.abs().max().item())


@pytest.mark.parametrize("a_trans,b_trans", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_majors(a_trans, b_trans, bn):
    assert run(256, 256, 512, a_trans, b_trans, bn=bn) < 3e-3


@pytest.mark.parametrize("shape", [(512, 512, 4096), (100, 72, 40), (16, 40, 32), (512, 16384, 512),
                                   (4096, 512, 512), (130, 260, 200)])
def test_shapes(shape):
    M, N, K = shape
    assert run(M, N, K, 0, 0) < 3e-3
    if M % 4 == 0:     # an M-major A needs a 16-byte row pitch
        assert run(M, N, K, 1, 0, bn=64) < 3e-3


@pytest.mark.parametrize("splits", [2, 4, 8])
@pytest.mark.parametrize("bn", [64, 256])
def test_split_k(splits, bn):
    assert run(512, 512, 8192, 0, 0, splits=splits, bn=bn) < 3e-3
    assert run(200, 300, 4000, 0, 1, splits=splits, bn=bn) < 3e-3   # ragged M: slices clip


@pytest.mark.parametrize("bn", [128, 256])
@pytest.mark.parametrize("a_trans,b_trans", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_cta_pair(bn, a_trans, b_trans):
    assert run(512, 1024, 512, a_trans, b_trans, bn=bn, pair=2) < 3e-3
    assert run(300, 2048, 700, a_trans, b_trans, bn=bn, pair=2) < 3e-3     # ragged M and K
    assert run(128, 512, 256, a_trans, b_trans, bn=bn, pair=2) < 3e-3      # empty second CTA rows
    assert run(512, 512, 8192, a_trans, b_trans, splits=4, bn=bn, pair=2) < 3e-3


@pytest.mark.parametrize("bn,pair", [(256, 2), (128, 2), (128, 1)])
@pytest.mark.parametrize("a_trans,b_trans", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_persistent_ws(bn, pair, a_trans, b_trans):
    """Persistent warp-specialised kernel (gemm_ws.cuh): several tiles per CTA,
    two TMEM accumulators, split-K slices and ragged edges."""
    ws = pair | 4
    assert run(512, 16384, 512, a_trans, b_trans, bn=bn, pair=ws) < 3e-3     # many tiles / CTA
    assert run(300, 2048, 700, a_trans, b_trans, bn=bn, pair=ws) < 3e-3      # ragged M and K
    assert run(128, 512, 256, a_trans, b_trans, bn=bn, pair=ws) < 3e-3
    assert run(512, 512, 8192, a_trans, b_trans, splits=18, bn=bn, pair=ws) < 3e-3
