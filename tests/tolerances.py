"""Stated parity tolerances (norm-wise max error ``||y - y_ref||_inf / ||y_ref||_inf``
against the float64 oracle), shared by the GPU parity tests.

Each family's bound sits at most ~10x above the largest error measured for it on
a B200 (``tests/golden/parity_errors_r2.json``, the ``CONVIO_PARITY_LOG`` record of
a full ``-m gpu`` run), so a precision regression in a split (3xTF32 / 3xF16) or a
dropped term fails the suite instead of hiding under a loose bound.  Bounds grow
like sqrt(C*R*S) (random-walk growth of an fp32 accumulation).
"""

# FP32 CUDA-core direct conv at the config-1 reduction length C*R*S = 576
# (measured max over the suite 9.2e-7, 2.4e-6 at C*R*S = 4608; SURVEY proposed 1e-5)
TOL_DIRECT = 5e-6


def _growth(c, r=3, s=3):
    return max(1.0, ((c * r * s) / 576) ** 0.5)


def tol_fp32(c, r=3, s=3):
    """FP32 FFMA direct conv."""
    return TOL_DIRECT * _growth(c, r, s)


def tol_3xtf32(c, r=3, s=3):
    """3xTF32 implicit GEMM (hi*lo + lo*hi + hi*hi, FP32 accumulate): the lo*lo term
    and the TF32 rounding of lo cost ~2^-21 per product (measured 5.8e-6 at C = 64,
    3.4e-5 at C = 512 with split-K partial sums)."""
    return 4 * tol_fp32(c, r, s)


# Winograd in FP32-level arithmetic (FFMA, 3xTF32 or 3xF16 element-wise GEMMs): the
# transforms amplify the fp32 rounding of V and U -- F(4,3)'s B^T entries up to 5
# and G's 1/6..1/24 -- so the bound is per e, grown with sqrt(C / 64).  Measured
# maxima: F(2,3) 6.7e-7 (C = 64), 2.0e-6 (C = 256); F(4,3) 6.7e-6 (C = 64),
# 1.3e-5 (C = 128), 1.9e-5 (C = 256), 1.9e-5 (C = 512, VGG-16 at batch 32).
# (Round 1 stated 1e-4 / 1e-3: up to 150x above the measured errors.)
TOL_WINO = {2: 5e-6, 4: 4e-5}


def tol_wino(e, c):
    return TOL_WINO[e] * max(1.0, (c / 64) ** 0.5)


# Reduced precision (stated, looser): TF32 / BF16 operands.  Measured maxima:
# TF32 implicit GEMM 8.4e-4, BF16 2.6e-3; tensor-core Winograd TF32 F(2,3) 8.8e-4,
# F(4,3) 8.3e-3, BF16 F(2,3) 3.6e-3, F(4,3) 6.0e-2 (the transforms amplify the
# operand rounding: F(4,3)'s B^T entries up to 5, G's down to 1/24)
TOL_TF32 = 5e-3
TOL_BF16 = 2e-2
TOL_WTC = {("tf32", 2): 5e-3, ("tf32", 4): 4e-2, ("bf16", 2): 3e-2, ("bf16", 4): 1.5e-1}


def tol_for(algorithm: str, c: int, e: int | None = None, r: int = 3) -> float:
    """Tolerance of one tuned plan (runner algorithm names)."""
    if algorithm in ("direct",):
        return tol_fp32(c, r, r)
    if algorithm in ("igemm_3xtf32", "igemm_3xf16"):
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
