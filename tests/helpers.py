"""Shared test helpers: the parity criterion and GPU availability."""
import numpy as np

TOL = 1e-5   # BASELINE.json north_star item 4: |R_gpu - R_ref| <= 1e-5 * sum_k |w_ik| |s_kj|


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def assert_parity(R_gpu: np.ndarray, R_ref: np.ndarray, T: np.ndarray, tol: float = TOL,
                  what: str = ""):
    """Element-wise |R_gpu - R_ref| <= tol * T (complex modulus, R5).

    Elements with T == 0 must be exact zeros.  Returns the worst |err| / T.
    """
    R_gpu = np.asarray(R_gpu)
    assert R_gpu.shape == R_ref.shape, (R_gpu.shape, R_ref.shape)
    assert np.isfinite(R_gpu.view(np.float32)).all(), f"{what}: non-finite output"
    err = np.abs(R_gpu.astype(np.complex128) - R_ref.astype(np.complex128))
    bad = err > tol * T
    if bad.any():
        idx = np.argwhere(bad)[0]
        raise AssertionError(
            f"{what}: {int(bad.sum())} elements out of tolerance; first at {tuple(idx)}: "
            f"gpu={R_gpu[tuple(idx)]} ref={R_ref[tuple(idx)]} err={err[tuple(idx)]:.3e} "
            f"T={T[tuple(idx)]:.3e}")
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(T > 0, err / np.where(T > 0, T, 1), 0.0)
    return float(rel.max()) if rel.size else 0.0


def assert_bitwise(a: np.ndarray, b: np.ndarray, what: str = ""):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    va, vb = a.view(np.uint32), b.view(np.uint32)
    if not np.array_equal(va, vb):
        idx = np.argwhere(va != vb)[0]
        raise AssertionError(f"{what}: bit patterns differ at {tuple(idx)}: "
                             f"{a.view(np.float32)[tuple(idx)]} vs {b.view(np.float32)[tuple(idx)]}")
