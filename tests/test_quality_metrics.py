"""Host-side metrics of the equal-budget quality harness: SSIM (Wang et al.
2004, uniform k x k windows) pinned to brute force over explicit windows and to the closed form for constant
images; MSE by definition."""
import numpy as np
import pytest

from paper_2406_16302_b200 import quality as Q


def _ssim_brute(img, ref, k):
    x, y = img.mean(axis=-1), ref.mean(axis=-1)
    L = float(y.max() - y.min()) or 1.0
    c1, c2 = (0.01 * L) ** 2, (0.03 * L) ** 2
    vals = []
    for i in range(x.shape[0] - k + 1):
        for j in range(x.shape[1] - k + 1):
            a, b = x[i:i + k, j:j + k].ravel(), y[i:i + k, j:j + k].ravel()
            ma, mb = a.mean(), b.mean()
            va, vb = ((a - ma) ** 2).mean(), ((b - mb) ** 2).mean()
            cab = ((a - ma) * (b - mb)).mean()
            vals.append(((2 * ma * mb + c1) * (2 * cab + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2)))
    return float(np.mean(vals))


@pytest.mark.parametrize("k", [3, 7])
def test_ssim_matches_explicit_windows(k):
    rng = np.random.default_rng(k)
    ref = rng.normal(size=(13, 17, 3))
    img = ref + 0.3 * rng.normal(size=ref.shape)
    assert abs(Q.ssim(img, ref, k) - _ssim_brute(img, ref, k)) < 1e-12


def test_ssim_identity_and_constant_closed_form():
    rng = np.random.default_rng(0)
    ref = rng.normal(size=(9, 9, 3))
    assert Q.ssim(ref, ref) == pytest.approx(1.0, abs=1e-12)
    # constant images a, b (variances 0): SSIM = (2ab + C1) / (a^2 + b^2 + C1); the range of a constant
    # reference is 0, so L = 1
    a, b = 0.25, -0.5
    c1 = 0.01 ** 2
    got = Q.ssim(np.full((8, 8, 3), a), np.full((8, 8, 3), b))
    assert got == pytest.approx((2 * a * b + c1) / (a * a + b * b + c1), rel=1e-12)


def test_ssim_decreases_with_noise():
    rng = np.random.default_rng(1)
    ref = rng.normal(size=(32, 32, 3))
    n = rng.normal(size=ref.shape)
    s = [Q.ssim(ref + e * n, ref) for e in (0.0, 0.1, 0.5, 2.0)]
    assert s[0] > s[1] > s[2] > s[3]


def test_mse_definition():
    a = np.arange(12.0).reshape(2, 2, 3)
    assert Q.mse(a, a + 2.0) == 4.0
