"""GPU calibration against the float64 oracle: hc_calib_svd (ΔW = W − deq, its SVD,
the rank-r factors U = P[:, :r], V = diag(σ)·Q[:, :r]ᵀ, P:142-145 / P:213-214, R4/R5) and
hc_calib_salience (φ, App. B.1 eq. A8).  Inputs: W ~ N(0, 0.02²) float32 quantised by the
oracle's RTN with bf16 scales, so both sides see the same canonical codes / scales / zeros."""
import numpy as np
import pytest
import torch

from oracle import allocate, factors
from oracle.packing import bf16_to_f64, f64_to_bf16_bits_rne
from oracle.quant import dequant, rtn_quantize

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hc():
    import paper_2605_05819_b200 as m
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return m


@pytest.fixture(scope="module")
def ctx(hc):
    return hc.Context(0)


def pack_rows(q: np.ndarray, bits: int) -> np.ndarray:
    """Canonical code stream (hcinfer.h, R1): element k of a row at bits [b·k, b·k + b)."""
    N, K = q.shape
    words = np.zeros((N, K * bits // 32), dtype=np.uint32)
    for n in range(N):
        acc = 0
        for k in range(K - 1, -1, -1):
            acc = (acc << bits) | int(q[n, k])
        for w in range(words.shape[1]):
            words[n, w] = (acc >> (32 * w)) & 0xFFFFFFFF
    return words


def calib_case(seed, M, N, K, bits, group=128):
    g = np.random.default_rng(seed)
    W = (0.02 * g.standard_normal((M, N, K))).astype(np.float32)
    codes, scales, zeros, dW = [], [], [], []
    for m in range(M):
        c, s = rtn_quantize(W[m].astype(np.float64), bits, group)
        q = (c + (1 << (bits - 1))).astype(np.int64)
        sb = f64_to_bf16_bits_rne(s)
        z = np.full((N, K // group), 1 << (bits - 1), dtype=np.uint8)
        codes.append(pack_rows(q, bits))
        scales.append(sb)
        zeros.append(z)
        dW.append(W[m].astype(np.float64) - dequant(q, bf16_to_f64(sb), z, group))   # ΔW = W − Ŵ
    return dict(W=W, codes=np.stack(codes), scales=np.stack(scales), zeros=np.stack(zeros), dW=dW, bits=bits,
                group=group)


def run_svd(ctx, case, r):
    M, N, K = case["W"].shape
    d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
    U = torch.zeros((M, N, r), dtype=torch.float64, device="cuda")
    V = torch.zeros((M, r, K), dtype=torch.float64, device="cuda")
    S = torch.zeros((M, min(N, K)), dtype=torch.float64, device="cuda")
    sweeps = ctx.calib_svd(d(case["W"], np.float32), d(case["codes"], np.int32), d(case["scales"], np.int16),
                           d(case["zeros"], np.uint8), case["bits"], case["group"], r, U, V, S)
    torch.cuda.synchronize()
    return U.cpu().numpy(), V.cpu().numpy(), S.cpu().numpy(), sweeps


@pytest.mark.parametrize("M,N,K,bits", [(3, 256, 384, 4), (2, 384, 256, 3), (1, 128, 512, 2), (2, 512, 128, 4)])
def test_svd_matches_oracle(ctx, M, N, K, bits):
    """σ within 1e-12·σ₁ of LAPACK's, the rank-r product U·V within 1e-10 of the oracle's, U orthonormal,
    the sign convention exact, and vector-wise agreement for the well-separated leading ranks; both the
    column (K <= N) and the row (K > N) orthogonalisation."""
    case = calib_case(10 + N + K + bits, M, N, K, bits)
    r = 32
    U, V, S, sweeps = run_svd(ctx, case, r)
    assert 1 <= sweeps < 40
    for m in range(M):
        Uo, Vo, so = factors.svd_factors(case["dW"][m], r)
        assert np.abs(S[m] - so).max() <= 1e-12 * so[0]
        assert np.all(np.diff(S[m]) <= 0)
        ref = Uo @ Vo
        assert np.abs(U[m] @ V[m] - ref).max() <= 1e-10 * np.abs(ref).max()
        assert np.abs(U[m].T @ U[m] - np.eye(r)).max() <= 1e-12
        for j in range(r):
            col = U[m][:, j]
            assert col[np.flatnonzero(col != 0.0)[0]] >= 0.0             # R5: first nonzero entry >= 0
        gaps = np.minimum(so[:r] - so[1:r + 1], np.concatenate([[np.inf], so[:r - 1] - so[1:r]]))
        ok = gaps > 1e-3 * so[0]
        assert np.abs(U[m][:, ok] - Uo[:, ok]).max() <= 1e-8
        assert np.abs(V[m][ok] - Vo[ok]).max() <= 1e-8 * so[0]


def test_full_rank_reconstructs_w(ctx):
    """Kept at full rank the factors reconstruct W: Ŵ + U·V = W (P:142 with r = min(N, K)), float64."""
    case = calib_case(77, 1, 256, 256, 3)
    U, V, S, _ = run_svd(ctx, case, 256)
    W = case["W"][0].astype(np.float64)
    W_hat = W - case["dW"][0]
    assert np.abs(W_hat + U[0] @ V[0] - W).max() <= 1e-13 * np.abs(W).max()


def test_eckart_young(ctx):
    """‖ΔW − U_r V_r‖_F² = Σ_{j>r} σ_j² for several r from one factorisation (rank-prefix)."""
    case = calib_case(78, 1, 384, 256, 4)
    U, V, S, _ = run_svd(ctx, case, 128)
    dW = case["dW"][0]
    for r in (8, 32, 128):
        res = dW - U[0][:, :r] @ V[0][:r]
        assert abs(np.sum(res * res) - np.sum(S[0][r:] ** 2)) <= 1e-10 * np.sum(S[0] ** 2)


def test_salience_bit_exact(ctx):
    """hc_calib_salience on the oracle's own σ (LAPACK) is bit-identical to oracle.allocate.salience; plus
    the SPEC worked example σ = (1, 0.9, 0.1, 0.05, 0.04) -> cut 3, φ = 14.8148... and the
    degenerate paths (n < 3, σ₁ = 0, flat spectrum -> φ = 1)."""
    specs = []
    for seed in range(6):
        case = calib_case(200 + seed, 1, 256, 256, 2 + seed % 3)
        specs.append(np.linalg.svd(case["dW"][0], compute_uv=False))
    g = np.random.default_rng(3)
    for _ in range(20):   # planted knees (synth-style spectra)
        c = g.uniform(2, 16)
        specs.append(np.exp(-np.arange(256) / c) + 0.05)
    specs.append(np.linspace(1.0, 0.5, 256))
    n = 256
    sig = torch.from_numpy(np.stack(specs)).cuda()
    phi = torch.zeros(len(specs), dtype=torch.float64, device="cuda")
    cut = torch.zeros(len(specs), dtype=torch.int32, device="cuda")
    ctx.calib_salience(sig, phi, cut)
    torch.cuda.synchronize()
    for i, s in enumerate(specs):
        o = allocate.salience(s)
        assert phi[i].item() == o.phi and int(cut[i].item()) == o.cut, (i, phi[i].item(), o.phi, cut[i].item(), o.cut)
    small = torch.tensor([[1.0, 0.9, 0.1, 0.05, 0.04], [0.0, 0.0, 0.0, 0.0, 0.0]], dtype=torch.float64, device="cuda")
    phi2 = torch.zeros(2, dtype=torch.float64, device="cuda")
    cut2 = torch.zeros(2, dtype=torch.int32, device="cuda")
    ctx.calib_salience(small, phi2, cut2)
    torch.cuda.synchronize()
    assert int(cut2[0].item()) == 3 and abs(phi2[0].item() - 14.814814814814815) <= 1e-12
    assert phi2[1].item() == 1.0 and int(cut2[1].item()) == 0


def test_calibrated_factors_drive_the_kernel(hc, ctx):
    """End to end: factors from hc_calib_svd, rounded to bf16, loaded with hc_load_layer; the decode kernel's
    output at rank r matches the oracle fed the same bf16 factors (2e-3), and at r = 64 it is closer to W·x
    than the uncompensated product (the compensation is real)."""
    from oracle import linear
    N, K, bits = 256, 512, 3
    case = calib_case(91, 1, N, K, bits)
    r = 64
    U, V, S, _ = run_svd(ctx, case, r)
    Ub, Vb = f64_to_bf16_bits_rne(U[0]), f64_to_bf16_bits_rne(V[0])
    x = f64_to_bf16_bits_rne(np.random.default_rng(4).standard_normal((1, K)))
    lc = dict(N=N, K=K, bits=bits, group=128, codes=case["codes"][0], scales=case["scales"][0], zeros=case["zeros"][0],
              U=Ub, V=Vb, x=x)
    L = 900
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
    ctx.load_layer([dict(layer=L, window=0, slot=0, N=N, K=K, bits=bits, codes=t(lc["codes"], np.int32),
                         scales=t(lc["scales"], np.int16).view(torch.bfloat16), zeros=t(lc["zeros"], np.uint8),
                         U=t(Ub, np.int16).view(torch.bfloat16), V=t(Vb, np.int16).view(torch.bfloat16),
                         r_stored=r, r_alloc=r)])
    y = torch.empty((1, N), dtype=torch.float32, device="cuda")
    ctx.compensated_linear(L, 0, t(x, np.int16).view(torch.bfloat16), y)
    torch.cuda.synchronize()
    yk = y.cpu().numpy()
    ref = linear.compensated_linear(lc, r)
    assert np.abs(yk - ref).max() <= 2e-3 * np.abs(ref).max()
    wx = bf16_to_f64(x) @ case["W"][0].astype(np.float64).T
    y0 = linear.compensated_linear(lc, 0)
    assert np.abs(yk - wx).max() < 0.8 * np.abs(y0 - wx).max()
