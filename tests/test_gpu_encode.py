"""GPU parity of the encode step itself: the
encode workspace written by ftgemm_encode, read back through the layout that
ftgemm_encode_layout reports, against the CPU oracle's Eq. (1) / Eq. (2)
checksums on the same seeded inputs.

* Ac_i[k], Br_j[k]: FP32 sums of FP32 / BF16 / TF32-truncated operands.  Integer
  inputs: exact.  Real inputs: within the a-priori bound of recursive FP32
  summation, |fl(sum x) - sum x| <= (n - 1) u sum |x| (u = 2^-24), n = tile width.
* B^r (tensor-core dtypes): the data columns are bit-exact copies of B, the
  three split columns sum exactly (in FP64) to the device's Br_j[k] and each is
  representable in the operand format, the last column of the slot is zero.
* Norms (threshold inputs, R1): relative 1e-5 against FP64.
Shapes cover several tiles, ragged M / N / K tails, odd and even numbers of
check-tile columns (the BF16 encode works on pairs of tiles), padded leading
dimensions and both tensor-core tile classes (BN = 256 and BN = 128)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import odt, padded

pytestmark = pytest.mark.gpu

U = 2.0 ** -24


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2305_01024_b200 import ftgemm as F
    F.lib()
    oracle.build()


def _operand_values(x: np.ndarray, dtype: str) -> np.ndarray:
    """The values the tensor core sees: TF32 drops the low 13 mantissa bits."""
    x = x.astype(np.float32)
    if dtype == "tf32":
        x = (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    return x


def _arr(ws, off, count, dt):
    return ws[off:off + count * np.dtype(dt).itemsize].cpu().numpy().view(dt) if count else np.zeros(0, dt)


SHAPES = [
    (300, 520, 200, None, None),        # ragged M / N, odd tile count (BN=128 class at this size)
    (1000, 1264, 704, None, None),      # 6 check-tile columns, last one 4 wide
    (777, 600, 520, 528, 608),          # padded leading dimensions, 3 tiles (odd), K tail
    (4096, 4096, 256, None, None),      # 128 x 256 instantiation: 17 tiles of 252
    (512, 8192, 1024, None, None),      # 33 tiles (odd) at the cfg3 width
]


@pytest.mark.parametrize("dist", ["signed", "int"])
@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32_simt"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s[:3])))
def test_encode_outputs(dtype, shape, dist):
    import torch
    from paper_2305_01024_b200 import ftgemm as F
    M, N, K, lda, ldb = shape
    A, B, _ = synth.problem(M, N, K, dist=dist, dtype=odt(dtype))
    g = F.FTGemm(dtype, M, N, K)
    p = g.plan
    L = F.encode_layout(dtype, M, N, K)
    g.enc_ws.fill_(0xA5)                 # stale bytes must be overwritten
    g.encode(padded(A, dtype, lda), padded(B, dtype, ldb))
    torch.cuda.synchronize()
    ws = g.enc_ws
    kp, tm, tn = L["kp"], p.check_tile_m, p.check_tile_n
    Av, Bv = _operand_values(A, dtype), _operand_values(B, dtype)

    # Eq. (1): Ac_i = e^T A_i ; Eq. (2): Br_j = B_j e   (oracle, FP64)
    ac_ref = oracle.encode_col(Av, tm)                    # [tiles_m][K]
    br_ref = oracle.encode_row(Bv, tn)                    # [tiles_n][K]
    ac = _arr(ws, L["ac"], p.tiles_m * kp, np.float32).reshape(p.tiles_m, kp).astype(np.float64)
    br = _arr(ws, L["br"], p.tiles_n * kp, np.float32).reshape(p.tiles_n, kp).astype(np.float64)
    assert np.all(ac[:, K:] == 0) and np.all(br[:, K:] == 0)
    absA = oracle.encode_col(np.abs(Av), tm)
    absB = oracle.encode_row(np.abs(Bv), tn)
    if dist == "int":
        assert np.array_equal(ac[:, :K], ac_ref) and np.array_equal(br[:, :K], br_ref)
    else:
        assert np.all(np.abs(ac[:, :K] - ac_ref) <= (tm - 1) * U * absA + 1e-30)
        assert np.all(np.abs(br[:, :K] - br_ref) <= (tn - 1) * U * absB + 1e-30)

    # norms
    A64, B64 = Av.astype(np.float64), Bv.astype(np.float64)
    rown = _arr(ws, L["rownorm"], M, np.float32)
    coln = _arr(ws, L["colnorm"], N, np.float32)
    acn = _arr(ws, L["acnorm"], p.tiles_m, np.float32)
    brn = _arr(ws, L["brnorm"], p.tiles_n, np.float32)
    np.testing.assert_allclose(rown, np.sqrt((A64 ** 2).sum(1)), rtol=1e-5)
    np.testing.assert_allclose(coln, np.sqrt((B64 ** 2).sum(0)), rtol=1e-5)
    np.testing.assert_allclose(acn, np.sqrt((ac_ref ** 2).sum(1)), rtol=1e-5)
    np.testing.assert_allclose(brn, np.sqrt((br_ref ** 2).sum(1)), rtol=1e-5)

    if dtype == "f32_simt":
        assert L["bt"] == -1
        return
    # the encoded operand B^r = [B_j, split(B_j e), 0]
    ld = L["bt_ld"]
    assert ld == p.tiles_n * p.bn and p.bn - tn == 4
    if dtype == "bf16":
        bt = _arr(ws, L["bt"], kp * ld, np.uint16).reshape(kp, ld)
        src = synth.f32_to_bf16_bits(B.astype(np.float32))
        val = lambda h: synth.bf16_bits_to_f32(h).astype(np.float64)   # noqa: E731
    else:
        bt = _arr(ws, L["bt"], kp * ld, np.uint32).reshape(kp, ld)
        src = B.astype(np.float32).view(np.uint32)
        val = lambda h: h.view(np.float32).astype(np.float64)          # noqa: E731
    for j in range(p.tiles_n):
        c0, c1 = j * tn, min(N, (j + 1) * tn)
        slot = bt[:K, j * p.bn:(j + 1) * p.bn]
        assert np.array_equal(slot[:, :c1 - c0], src[:, c0:c1]), j
        assert np.all(slot[:, c1 - c0:tn] == 0), j
        parts = val(slot[:, tn:tn + 3])
        assert np.array_equal(parts.sum(1), br[j, :K]), j          # exact three-term split
        assert np.all(slot[:, tn + 3] == 0), j
        if dtype == "tf32":                                         # hi, mid: TF32-representable
            assert np.all((slot[:, tn:tn + 2] & 0x1FFF) == 0), j
    assert np.all(bt[K:] == 0)
    # the split rows of e^T A_i, pre-swizzled as MMA rows 125..127
    nkb = kp // p.bk
    y = _arr(ws, L["y"], p.tiles_m * nkb * 384, np.uint8).reshape(p.tiles_m, nkb, 3, 8, 16)
    for r in range(3):
        perm = [c ^ ((125 + r) & 7) for c in range(8)]
        rows = y[:, :, r][:, :, perm].reshape(p.tiles_m, nkb * 128)
        if dtype == "bf16":
            terms = synth.bf16_bits_to_f32(rows.copy().view(np.uint16)).astype(np.float64)
        else:
            terms = rows.copy().view(np.float32).astype(np.float64)
        total = terms if r == 0 else total + terms
    assert np.array_equal(total, ac)                                # exact three-term split of Ac


@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32_simt"])
@pytest.mark.parametrize("shape", [SHAPES[1], SHAPES[2], SHAPES[4]], ids=lambda s: "x".join(map(str, s[:3])))
def test_encode_one_launch_equals_per_operand(dtype, shape):
    """Both operands in one launch (encode_ab_kernel, which = 3) write the same
    bytes as the per-operand kernels (which = 1, then which = 2): the same
    per-block arithmetic, only the block-index mapping differs."""
    import torch
    from paper_2305_01024_b200 import ftgemm as F
    M, N, K, lda, ldb = shape
    A, B, _ = synth.problem(M, N, K, dist="signed", dtype=odt(dtype))
    Ad, Bd = padded(A, dtype, lda), padded(B, dtype, ldb)
    g = F.FTGemm(dtype, M, N, K)
    L = F.encode_layout(dtype, M, N, K)
    p = g.plan
    g.enc_ws.fill_(0x5A)
    g.encode(Ad, Bd)
    one = g.enc_ws.clone()
    g.enc_ws.fill_(0xC3)
    g.encode(Ad, None, which=1)
    g.encode(None, Bd, which=2)
    torch.cuda.synchronize()
    two = g.enc_ws
    kp = L["kp"]
    regions = [("ac", p.tiles_m * kp * 4), ("br", p.tiles_n * kp * 4), ("rownorm", M * 4), ("colnorm", N * 4),
               ("acnorm", p.tiles_m * 4), ("brnorm", p.tiles_n * 4)]
    if dtype != "f32_simt":
        regions += [("bt", kp * L["bt_ld"] * (2 if dtype == "bf16" else 4)), ("y", p.tiles_m * (kp // p.bk) * 384)]
    for name, nbytes in regions:
        o = L[name]
        assert torch.equal(one[o:o + nbytes], two[o:o + nbytes]), name
