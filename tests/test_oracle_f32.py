"""Pins for the single-precision oracle (NEXT-4; the paper's experiments are single
precision, and it 'tested ... both single precision and double
precision').  The FP32 listings are pinned to the (pinned) FP64
oracle within binary32 error bounds, to SPEC.md examples, and to binary32
arithmetic itself."""
import numpy as np

import oracle
import synth

U32 = 2.0 ** -24


def test_f32_spec_examples():
    x, h, r = oracle.cg_f32(np.eye(3), [1.0, -2.0, 3.0], tol=1e-6)
    assert r.converged and r.iterations == 1 and x.tolist() == [1.0, -2.0, 3.0]
    x, h, r = oracle.cg_f32(np.diag([1.0, 2.0, 3.0]), np.ones(3), tol=1e-6)
    assert r.converged and r.iterations <= 3
    assert np.allclose(x, [1.0, 0.5, 1.0 / 3.0], rtol=4 * U32, atol=0)
    x, h, r = oracle.bicgstab_f32(np.array([[2.0, 1.0], [0.0, 3.0]]), [3.0, 3.0], tol=1e-6)
    assert r.converged and np.allclose(x, [1.0, 1.0], rtol=4 * U32, atol=0)
    assert x.dtype == np.float32


def test_f32_is_binary32_arithmetic():
    """1e8f + 1 - 1e8f: sequential float sums lose the 1 (float spacing at 1e8
    is 8); a double evaluation would keep it -> the listing really runs in float."""
    A = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    b = np.array([1e8, 1.0, -1e8], dtype=np.float32)
    x, h, r = oracle.cg_f32(A, b, tol=0.0, maxit=1)
    assert x.tolist() == [1e8, 1.0, -1e8]
    # ||b||^2 in float: 1e16 + 1 + 1e16 == 2e16 exactly in float arithmetic
    assert np.float32(1e8) * np.float32(1e8) + np.float32(1.0) == np.float32(1e16)


def test_f32_cg_vs_f64_oracle():
    """Attainable accuracy of FP32 CG ~ kappa * u32: at kappa = 1e3, tol 1e-5 the
    FP32 solution is within 1e3 * 2^-24 * 10 of the FP64 one; the first
    residuals agree to a few u32 * sqrt(n); counts within 2."""
    for n, kappa in [(1024, 1e3), (2048, 1e2)]:
        A, c, b = synth.gspd(n, kappa)
        x32, h32, r32 = oracle.cg_f32(A, b, tol=1e-5)
        x64, h64, r64 = oracle.cg(A, b, tol=1e-5)
        assert r32.converged and abs(r32.iterations - r64.iterations) <= 2
        assert np.linalg.norm(x32 - x64) <= 10 * kappa * U32 * np.linalg.norm(x64)
        assert np.all(np.abs(h32[:5] - h64[:5]) <= 100 * U32 * h64[:5])


def test_f32_bicgstab_vs_f64_oracle():
    for n, kd in [(1024, 4), (1024, 16), (4096, 16)]:
        A, b = synth.gdd(n, kd)
        x32, h32, r32 = oracle.bicgstab_f32(A, b, tol=1e-5)
        x64, h64, r64 = oracle.bicgstab(A, b, tol=1e-5)
        assert r32.converged and abs(r32.iterations - r64.iterations) <= 2
        assert np.linalg.norm(x32 - x64) <= 10 * 1.03 * kd * U32 * np.linalg.norm(x64) + 1e-5 * np.linalg.norm(x64)
        assert oracle.true_relres_ld(A, b, x32.astype(np.float64)) <= 10 * 1e-5
