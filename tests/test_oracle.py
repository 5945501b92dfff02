"""CPU tests pinning the oracle (oracle/lc_oracle.c) before it is trusted:
SPEC.md known-answer vectors + the reference-generated fixtures in
tests/golden/ (+ live cross-checks against oracle/_ref when it is built)."""
import numpy as np
import pytest

from conftest import golden
from oracle.oracle import rel_l2


# ---------------------------------------------------------------- SPEC KATs
def test_spec_dft_vector(lc):
    want = np.array([10, -2 + 2j, -2, -2 - 2j])
    np.testing.assert_allclose(lc.dft_naive([1, 2, 3, 4]), want, atol=1e-12)
    np.testing.assert_allclose(lc.apply_plan([1, 2, 3, 4], r=2), want, atol=1e-12)
    np.testing.assert_allclose(lc.dft_naive(want, inverse=True), [1, 2, 3, 4], atol=1e-12)


def test_spec_convolutions(lc):
    u, k = [1, 2, 3, 4], [1, 1, 0, 0]
    np.testing.assert_allclose(lc.conv_naive_real(u, k, causal=False), [5, 3, 5, 7])
    np.testing.assert_allclose(lc.conv_naive_real(u, k, causal=True), [1, 3, 5, 7])
    np.testing.assert_allclose(lc.conv_butterfly(u, k, causal=False).real, [5, 3, 5, 7], atol=1e-12)
    np.testing.assert_allclose(lc.conv_butterfly(u, k, causal=True).real, [1, 3, 5, 7], atol=1e-12)
    np.testing.assert_allclose(lc.conv_real_packed(u, k, causal=False), [5, 3, 5, 7], atol=1e-12)


def test_spec_three_pass_example(lc):
    u = np.arange(1, 9, dtype=float)
    k = np.array([1, 1, 0, 0, 0, 0, 0, 0], dtype=float)
    y = lc.conv_three_pass(u, k, 4, 2)
    np.testing.assert_allclose(y.real, [9, 3, 5, 7, 9, 11, 13, 15], atol=1e-12)
    np.testing.assert_allclose(y.real, lc.conv_naive_real(u, k, causal=False), atol=1e-12)


def test_spec_regularizers(lc):
    np.testing.assert_allclose(lc.squash([0.5, -0.3, 0.1], 0.2), [0.3, -0.1, 0.0], atol=1e-15)
    np.testing.assert_allclose(lc.smooth([1, 1, 1], 1), [2 / 3, 1, 2 / 3])
    np.testing.assert_allclose(lc.smooth([3, -1, 2], 0), [3, -1, 2])


def test_spec_geometric_envelope(lc):
    # position 0 has envelope 1: geometric K[h,0] equals the raw normal draw
    H, N = 5, 32
    K, _ = lc.init_kernels(1, H, N, 11)
    Kr, _ = lc.init_kernels(0, H, N, 11)
    np.testing.assert_array_equal(K[:, 0], Kr[:, 0])
    h, i = 3, 17
    dec = (H / 2) ** (h / H)
    np.testing.assert_allclose(K[h, i], Kr[h, i] * np.exp(-(i / N) * dec), rtol=1e-14)


def test_spec_identity_and_skip_layers(lc):
    B, H, N = 2, 3, 16
    u = lc.signal_batch(1, B, H, N)
    K = np.zeros((H, N))
    K[:, 0] = 1.0
    y = lc.regularized_long_conv(u, K, np.zeros(H), 0.0, 0)
    np.testing.assert_allclose(y, u, atol=1e-13)
    D = np.array([0.5, -2.0, 3.0])
    y = lc.regularized_long_conv(u, np.full((H, N), 0.1), D, lam=10.0, p=0)
    np.testing.assert_allclose(y, D[None, :, None] * u, atol=1e-13)


def test_spec_learned_identities(lc):
    n = 64
    x = np.random.default_rng(1).standard_normal(n) + 0j
    bl = lc.learned_init(n, 4)
    np.testing.assert_allclose(lc.learned_forward(bl, x, 4), lc.apply_plan(x, r=4), atol=1e-12)
    assert np.all(lc.learned_forward(np.zeros_like(bl), x, 4) == 0)


def test_learned_finite_difference(lc):  # SPEC.md:254 (n=8, r=2, tol 1e-6)
    rng = np.random.default_rng(11)
    n = 8
    bl = lc.learned_init(n, 2) + 0.3 * (rng.standard_normal(12) + 1j * rng.standard_normal(12))
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    g = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    J = lambda b, xx: np.real(np.vdot(g, lc.learned_forward(b, xx, 2)))  # noqa: E731
    db, dx = lc.learned_gradients(bl, x, g, 2)
    eps = 1e-6
    for i in range(bl.size):
        for d, comp in ((1.0, "re"), (1j, "im")):
            bp, bm = bl.copy(), bl.copy()
            bp[i] += eps * d
            bm[i] -= eps * d
            fd = (J(bp, x) - J(bm, x)) / (2 * eps)
            an = db[i].real if comp == "re" else db[i].imag
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an))


def test_backward_finite_difference(lc):
    rng = np.random.default_rng(3)
    B, H, N = 2, 2, 16
    u = rng.standard_normal((B, H, N))
    dy = rng.standard_normal((B, H, N))
    Kb = rng.standard_normal((H, N))
    D = rng.standard_normal(H)
    du, dK, dD = lc.long_conv_backward(u, dy, Kb, D)
    L = lambda uu, kk, dd: np.sum(dy * lc.long_conv_forward(uu, kk, dd))  # noqa: E731
    eps = 1e-6
    for idx in [(0, 0, 3), (1, 1, 15), (0, 1, 0)]:
        up, um = u.copy(), u.copy()
        up[idx] += eps
        um[idx] -= eps
        assert abs((L(up, Kb, D) - L(um, Kb, D)) / (2 * eps) - du[idx]) < 1e-6
    for idx in [(0, 0), (1, 7), (1, 15)]:
        kp, km = Kb.copy(), Kb.copy()
        kp[idx] += eps
        km[idx] -= eps
        assert abs((L(u, kp, D) - L(u, km, D)) / (2 * eps) - dK[idx]) < 1e-6
    dp = D.copy()
    dp[1] += eps
    dm = D.copy()
    dm[1] -= eps
    assert abs((L(u, Kb, dp) - L(u, Kb, dm)) / (2 * eps) - dD[1]) < 1e-6


# ------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("name", ["layer_b1h1n1024", "layer_b3h4n256", "layer_b2h2n128_circ",
                                  "layer_b2h3n64_drop"])
def test_golden_layer(lc, name):
    g = golden(name)
    causal, training = bool(g["causal"]), bool(g["training"])
    Kbar = lc.regularize_bank(g["K"], float(g["lam"]), int(g["p"]), float(g["rate"]), 0,
                              int(g["seed"]), training)
    np.testing.assert_array_equal(Kbar, g["Kbar"])
    y = lc.regularized_long_conv(g["u"], g["K"], g["D"], float(g["lam"]), int(g["p"]),
                                 float(g["rate"]), 0, int(g["seed"]), causal, training)
    for key in [k for k in g if k.startswith("y_engine")]:
        assert rel_l2(y, g[key]) < 1e-13, key
    if causal:
        du, dKbar, dD = lc.long_conv_backward(g["u"], g["dy"], Kbar, g["D"], causal)
        assert rel_l2(du, g["du"]) < 1e-13
        assert rel_l2(dKbar, g["dKbar"]) < 1e-13
        assert rel_l2(dD, g["dD"]) < 1e-13
        dK = lc.regularizer_backward(g["K"], float(g["lam"]), int(g["p"]), dKbar,
                                     float(g["rate"]), int(g["seed"]), training)
        assert rel_l2(dK, g["dK"]) < 1e-13


def test_golden_transforms(lc):
    g = golden("apply_plan_8192")
    assert lc.plan_factors(8192) == list(g["factors"]) == [16, 16, 16, 2]
    np.testing.assert_array_equal(lc.apply_plan(g["x"]), g["fwd"])
    np.testing.assert_array_equal(lc.apply_plan(g["x"], inverse=True), g["inv"])
    g = golden("apply_plan_96_r16")
    assert lc.plan_factors(96) == list(g["factors"])
    np.testing.assert_array_equal(lc.apply_plan(g["x"]), g["fwd"])


def test_golden_three_pass(lc):
    g = golden("three_pass_4096")
    l, m = int(g["l"]), int(g["m"])
    assert int(g["sweeps"]) == 3  # SPEC.md:330 (Proposition 1)
    np.testing.assert_array_equal(lc.three_pass_dk(g["k"], l, m), g["dk"])
    assert rel_l2(lc.conv_three_pass(g["u"], g["k"], l, m), g["y"]) < 1e-14


def test_golden_real_packed(lc):
    g = golden("real_packed_512")
    np.testing.assert_array_equal(lc.conv_real_packed(g["u"], g["k"], True), g["causal"])
    np.testing.assert_array_equal(lc.conv_real_packed(g["u"], g["k"], False), g["circular"])


@pytest.mark.parametrize("name,r", [("learned_1024", 16), ("learned_64_r4", 4)])
def test_golden_learned(lc, name, r):
    g = golden(name)
    np.testing.assert_array_equal(lc.learned_forward(g["blocks"], g["x"], r), g["y"])
    db, dx = lc.learned_gradients(g["blocks"], g["x"], g["g"], r)
    np.testing.assert_array_equal(db, g["dblocks"])
    np.testing.assert_array_equal(dx, g["dx"])


def test_golden_regularizers_and_rng(lc):
    g = golden("regularizers_64")
    np.testing.assert_array_equal(lc.squash(g["k"], 0.2), g["squash"])
    np.testing.assert_array_equal(lc.smooth(g["k"], 2), g["smooth"])
    assert rel_l2(lc.smooth_frequency(g["k"], 2), g["smooth_freq"]) < 1e-13
    g = golden("rng")
    np.testing.assert_array_equal(lc.normal_draws(1, 0, 16), g["normal"])
    np.testing.assert_array_equal(lc.uniform_draws(7, 3, 16), g["uniform"])


# --------------------------------------------- live cross-check vs _ref
def test_live_reference_agreement(lc, ref):
    B, H, N = 2, 3, 8  # SPEC.md:458 (engines agree within 1e-9 at B=2,H=3,N=8, seed 17)
    u = lc.signal_batch(17, B, H, N)
    K, D = lc.init_kernels(0, H, N, 17)
    y = lc.regularized_long_conv(u, K, D, 0.01, 1)
    for e in (0, 1, 2):
        assert np.abs(ref.regularized_long_conv(u, K, D, 0.01, 1, engine=e) - y).max() < 1e-9
    u = lc.signal_batch(1, 2, 4, 2048)
    K, D = lc.init_kernels(1, 4, 2048, 3)
    assert rel_l2(lc.regularized_long_conv(u, K, D, 0.003, 1),
                  ref.regularized_long_conv(u, K, D, 0.003, 1)) < 1e-14
