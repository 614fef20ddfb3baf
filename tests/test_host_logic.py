"""Host-side logic of the CUDA path that can be checked without a GPU, against the oracle."""
import numpy as np
import pytest

import oracle


def _screen_constants(T):
    """The constants launch_enc_fwd derives (csrc/k_encoder.cu): the no-fire bound thr (fp32, rounded
    down) and the spikes-only screen's zskip (fp32, rounded up)."""
    thr64 = 1.0 / (T * (1.0 + T * 2.0 ** -22))
    thr = np.float32(thr64)
    if float(thr) > thr64:
        thr = np.nextafter(thr, np.float32(0))
    zs64 = (-np.log(float(thr)) + 1e-6) * (1.0 + 1e-6)
    zskip = np.float32(zs64)
    if float(zskip) < zs64:
        zskip = np.nextafter(zskip, np.float32(np.inf))
    return thr, zskip


@pytest.mark.parametrize("T", [1, 5, 16, 33])
def test_spikes_only_screen_never_drops_a_spike(T):
    """enc_fwd_kernel's spikes-only screen skips an element when its fp32 z32 = RN(RN(d32 d32) inv32)
    (d32 = RN(s - mu), inv32 = RN32(1 / (2 sigma^2))) exceeds zskip. Claim: every skipped element has
    oracle A < thr, so the oracle's encoder gives it no spike at any step. Checked by brute force on
    a wide random spread of s / mu / sigma and on adversarial points placed within a few ulp of the
    screen's boundary."""
    thr, zskip = _screen_constants(T)
    rng = np.random.default_rng(T)
    n = 200_000
    s = rng.normal(0, 3, n).astype(np.float32)
    mu = rng.normal(0, 3, n).astype(np.float32)
    sg = np.exp(rng.uniform(np.log(1e-3), np.log(30.0), n)).astype(np.float32)
    # adversarial: |s - mu| placed so that z sits at zskip (1 +- a few 1e-7)
    m = 100_000
    mu2 = rng.normal(0, 3, m).astype(np.float32)
    sg2 = np.exp(rng.uniform(np.log(1e-2), np.log(3.0), m)).astype(np.float32)
    d2 = np.sqrt(float(zskip) * 2.0 * sg2.astype(np.float64) ** 2) * (1.0 + rng.uniform(-4e-7, 4e-7, m))
    s2 = (mu2.astype(np.float64) + np.where(rng.random(m) < 0.5, -d2, d2)).astype(np.float32)
    s, mu, sg = np.concatenate([s, s2]), np.concatenate([mu, mu2]), np.concatenate([sg, sg2])
    # the kernel's screen, in IEEE fp32 (numpy float32 arithmetic rounds to nearest even)
    den = 2.0 * (sg.astype(np.float64) ** 2)
    inv32 = (1.0 / den).astype(np.float32)
    d32 = (s - mu).astype(np.float32)
    z32 = (d32 * d32).astype(np.float32) * inv32
    skipped = z32 > zskip
    assert skipped.sum() > 0 and (~skipped).sum() > 0
    # oracle A for each (s, mu, sigma) triple: one observation dim, one encoder neuron per element
    A = np.empty(s.shape[0], np.float32)
    for lo in range(0, s.shape[0], 50_000):
        hi = min(lo + 50_000, s.shape[0])
        k = np.arange(hi - lo)
        # gaussian_stim takes s [B][S] and (mu, sigma) [S][E]: B = 1 row, S elements, E = 1
        A[lo:hi] = oracle.gaussian_stim(s[None, lo:hi], mu[lo:hi, None], sg[lo:hi, None])[0, k]
    assert np.all(A[skipped] < thr), "a skipped element reaches the no-fire bound"
    spikes = oracle.encode_spikes(A[None, skipped], T)
    assert not spikes.any(), "a skipped element fires"
