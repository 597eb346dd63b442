"""Stated parity tolerances (norm-wise max error ``||y - y_ref||_inf / ||y_ref||_inf``
against the float64 oracle), shared by the GPU parity tests.

Each family's bound sits at most ~10x above the largest error measured for it on
a B200 (``tests/golden/parity_errors_r2.json``, the ``CONVIO_PARITY_LOG`` record of
a full ``-m gpu`` run), so a precision regression in a split (3xTF32 / 3xF16) or a
dropped term fails the suite instead of hiding under a loose bound.  Bounds grow
like sqrt(C*R*S) (random-walk growth of an fp32 accumulation).
"""

# FP32 CUDA-core direct conv at the config-1 reduction length C*R*S = 576
# (measured max over the suite 6.1e-7; SURVEY's proposal was 1e-5)
TOL_DIRECT = 1e-5


def _growth(c, r=3, s=3):
    return max(1.0, ((c * r * s) / 576) ** 0.5)


def tol_fp32(c, r=3, s=3):
    """FP32 FFMA direct conv."""
    return TOL_DIRECT * _growth(c, r, s)


def tol_3xtf32(c, r=3, s=3):
    """3xTF32 implicit GEMM (hi*lo + lo*hi + hi*hi, FP32 accumulate): the lo*lo term
    and the TF32 rounding of lo cost ~2^-21 per product, like an fp32 rounding."""
    return 2 * tol_fp32(c, r, s)


# Winograd in FP32-level arithmetic (FFMA, 3xTF32 or 3xF16 element-wise GEMMs): the
# transforms amplify the fp32 rounding of V and U -- F(4,3)'s B^T entries up to 5
# and G's 1/6..1/24 -- so the bound is per e, grown with sqrt(C / 64)
TOL_WINO = {2: 1e-4, 4: 1e-3}


def tol_wino(e, c):
    return TOL_WINO[e] * max(1.0, (c / 64) ** 0.5)


# Reduced precision (stated, looser): TF32 / BF16 operands
TOL_TF32 = 5e-3
TOL_BF16 = 3e-2
TOL_WTC = {("tf32", 2): 5e-3, ("tf32", 4): 2e-2, ("bf16", 2): 5e-2, ("bf16", 4): 1.5e-1}


def tol_for(algorithm: str, c: int, e: int | None = None, r: int = 3) -> float:
    """Tolerance of one tuned plan (runner algorithm names)."""
    if algorithm in ("direct",):
        return tol_fp32(c, r, r)
    if algorithm == "igemm_3xtf32":
        return tol_3xtf32(c, r, r)
    if algorithm == "igemm_tf32":
        return TOL_TF32
    if algorithm == "igemm_bf16":
        return TOL_BF16
    if algorithm in ("winograd", "winograd_nhwc", "winograd_tc_3xtf32", "winograd_tc_3xf16"):
        return tol_wino(e, c)
    if algorithm.startswith("winograd_tc_"):
        return TOL_WTC[(algorithm[len("winograd_tc_"):], e)]
    raise KeyError(algorithm)
