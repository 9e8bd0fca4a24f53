"""Pins of the oracle's reduced-precision storage (a4 / O5): IEEE 754 RNE
conversions (P:151 ref 26) against numpy/torch conversions and
the SPEC's worked examples, and the diagonal mass fix-up (reading A10)."""
import numpy as np
import pytest
import torch

import fdirw_inputs as fi


def test_spec_rounding_examples(oracle_lib):
    o = oracle_lib
    assert o.round_fmt(1.0, "fp16") == 1.0
    assert o.round_fmt(1.0 + 2 ** -11, "fp16") == 1.0          # S:397 tie → even
    assert o.round_fmt(1.0 + 3 * 2 ** -11, "fp16") == 1.0 + 2 ** -9  # tie → even (up)
    assert o.round_fmt(65520.0, "fp16") == float("inf")        # S:398 overflow tie
    assert o.round_fmt(65504.0, "fp16") == 65504.0
    assert o.round_fmt(0.5, "fp32") == 0.5
    assert o.round_fmt(1.0 + 2 ** -24, "fp32") == 1.0           # S:405 tie → even
    assert o.round_fmt(3.4e38 * 1.1, "fp32") == float("inf")
    assert o.round_fmt(1.0 + 2 ** -8, "bf16") == 1.0            # bf16 tie → even
    assert o.round_fmt(1.0 + 3 * 2 ** -8, "bf16") == 1.0 + 2 ** -6
    assert o.round_fmt(2 ** -24, "fp16") == 2 ** -24            # smallest fp16 subnormal
    assert o.round_fmt(2 ** -25, "fp16") == 0.0                 # tie → even (0)
    assert o.round_fmt(1.5 * 2 ** -25, "fp16") == 2 ** -24


def _corpus(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    mags = 10.0 ** rng.uniform(-45, 39, n)
    x = (mags * rng.choice([-1.0, 1.0], n)).astype(np.float32)
    # add exact ties and boundary values
    extra = np.array([0.0, -0.0, 1.0, 65504, 65520, 65519.99, 6.1035156e-05, 5.9604645e-08, 2.9802322e-08,
                      1.0009765625, 1.00048828125, 3.0517578e-05, 1.1754944e-38, 3.3895314e38, 3.4028235e38],
                     np.float32)
    return np.concatenate([x, extra, -extra])


def test_f16_matches_numpy(oracle_lib):
    x = _corpus(100_000, 1)
    ref = x.astype(np.float16).view(np.uint16)
    got = np.array([oracle_lib.f32_to_f16_bits(float(v)) for v in x], np.uint16)
    np.testing.assert_array_equal(got, ref)


def test_bf16_matches_torch(oracle_lib):
    x = _corpus(100_000, 2)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = np.array([oracle_lib.f32_to_bf16_bits(float(v)) for v in x], np.uint16)
    np.testing.assert_array_equal(got, ref)


def test_fp64_to_fp32_matches_numpy(oracle_lib):
    rng = np.random.Generator(np.random.PCG64(3))
    x = rng.standard_normal(20000) * 10.0 ** rng.uniform(-30, 30, 20000)
    got = np.array([oracle_lib.round_fmt(float(v), "fp32") for v in x])
    np.testing.assert_array_equal(got, x.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("fmt", ["fp32", "fp16", "bf16"])
def test_quantize_mass_fix(oracle_lib, fmt):
    """A10 (round 2): off-centre weights are RNE_fmt(RNE_fp32(W)); the diagonal is the fp32
    pair (hi, lo) of d = 1 − Σ_{o≠0} W̃, so every stored column sums to 1 within ~2^-48 (an
    fp32 diagonal alone: half an fp32 ulp, 3e-8, biased per class of identical windows)."""
    mask = fi.random_two_phase((8, 7, 6), 0.6, seed=1)
    pb = oracle_lib.Problem(mask=mask, dh=1.0, D_fast=1.0, D_slow=1e-3, dt=0.1 * 30, R=2)
    W = oracle_lib.build_kernels(pb)
    Wq = oracle_lib.quantize(pb, W, fmt)
    c = pb.K // 2
    off = np.ones(pb.K, bool)
    off[c] = False
    conv = {"fp32": lambda a: a.astype(np.float32).astype(np.float64),
            "fp16": lambda a: a.astype(np.float32).astype(np.float16).astype(np.float64),
            "bf16": lambda a: torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).double().numpy()}[fmt]
    np.testing.assert_array_equal(Wq[..., off], conv(W[..., off]))
    diag = Wq[..., c]
    hi = diag.astype(np.float32).astype(np.float64)
    lo = diag - hi
    assert np.all(lo == lo.astype(np.float32))                # an fp32 pair: hi + lo exactly
    assert np.all(np.abs(lo) <= np.abs(hi) * 2.0 ** -24)      # lo below half an ulp of hi
    col = Wq.sum(-1)
    np.testing.assert_allclose(col, 1.0, rtol=0, atol=1e-14)
    d = 1.0 - (Wq[..., off]).sum(-1)                          # the exact fix-up value
    assert np.abs(diag - d).max() <= 2.0 ** -47 * np.abs(d).max()
    if fmt == "fp32":  # (fp16 sums are often exact in fp32; fp32 weights' are not)
        assert np.abs(hi - d).max() > 1e-10                   # an fp32 diagonal alone would miss it
    # without the fix-up, the column sum drifts by the storage format's rounding
    Wn = oracle_lib.quantize(pb, W, fmt, mass_fix=False)
    if fmt == "bf16":
        assert np.abs(Wn.sum(-1) - 1).max() > 1e-4


def test_fp16_underflow_absorbed(oracle_lib):
    """A14: fp16 flushes tail weights below 2^-25 to 0; the fix-up keeps mass."""
    mask = fi.random_two_phase((9, 9, 9), 0.5, seed=6)
    pb = oracle_lib.Problem(mask=mask, dh=1.0, D_fast=1.0, D_slow=1e-5, dt=0.1 * 200, R=3)
    W = oracle_lib.build_kernels(pb, (3, 6, 3, 6, 3, 6))
    Wq = oracle_lib.quantize(pb, W, "fp16")
    nz_before = np.count_nonzero(W)
    nz_after = np.count_nonzero(Wq)
    assert nz_after < nz_before
    np.testing.assert_allclose(Wq.sum(-1), 1.0, atol=1e-14)
