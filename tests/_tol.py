"""Comparison rules of SURVEY.md §8(c) C8 (the north star's tolerances made precise),
shared by the GPU parity tests."""
import numpy as np

TOL_U, TOL_C, TOL_G = 1e-9, 1e-10, 1e-7


def component_err(got, ref, floor_frac=1e-3):
    """max_i |got_i - ref_i| / max(|ref_i|, floor_frac * |ref|_inf): the per-component
    gradient rule, with the floor for near-zero entries."""
    got, ref = np.asarray(got, float).ravel(), np.asarray(ref, float).ravel()
    scale = np.abs(ref).max() if ref.size else 0.0
    if scale == 0.0:
        return float(np.abs(got).max()) if got.size else 0.0
    return float((np.abs(got - ref) / np.maximum(np.abs(ref), floor_frac * scale)).max())


def assert_components(got, ref, tol=TOL_G, what=""):
    e = component_err(got, ref)
    assert e <= tol, f"{what} per-component error {e:.3e} > {tol:.0e}"
