"""CPU restatement of the reference's convolution semantics (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline -- never as a product code path.

The reference package never computes a convolution value; its semantics live
in the DAG builders:

* direct: ``y[b,oc,oy,ox] = sum_c sum_ky sum_kx x[b,c,oy*mu+ky,ox*mu+kx] * w[oc,c,ky,kx]``
  as one left-deep sum in ``(c, ky, kx)`` order over a pre-padded input
  (``pkg/src/convio/dag.py:270-284``; padding is geometry preprocessing,
  ``model.py:65-70``);
* Winograd: per (b, oc, tile): ``P = B^T d B`` and ``J = G g G^T`` per channel
  (step 1), ``Lambda = P . J`` (step 2), ``Pi = sum_c Lambda`` left-deep over
  ``c`` (step 3), ``y = A^T Pi A`` (step 4) (``dag.py:343-401``); outputs not
  divisible by ``e`` are computed on the padded domain
  (``dag.py:291-299``) and cropped.

Everything is float64.  Parity status: **pinned to the reference's own code**.
The reference ships no conv value, but its direct-convolution DAG fixes every
arithmetic step, so ``tests/golden/make_dag_golden.py`` evaluates the
REFERENCE's ``build_direct_conv_dag`` vertex by vertex on seeded inputs (11
shapes: strides 1-3, 1x1 / 3x3 / 5x5 / 3x2 kernels, batch 2) and
``tests/test_dag_parity.py`` requires :func:`direct_conv` and the C
restatement to reproduce those values bit for bit; the Winograd tiling
(:func:`tile_patches`) is checked against the patch leaves of the reference's
``build_winograd_dag``.  Cross-checks: the direct path against
``torch.nn.functional.conv2d`` in float64, the Winograd path against the
direct path (~1e-12), the C restatement against both (``tests/test_oracle.py``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import winograd_mats

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libconv_oracle.so")


def pad_input(x: np.ndarray, padding: int) -> np.ndarray:
    if padding == 0:
        return np.asarray(x, dtype=np.float64)
    return np.pad(np.asarray(x, dtype=np.float64),
                  ((0, 0), (0, 0), (padding, padding), (padding, padding)))


def direct_conv(x: np.ndarray, w: np.ndarray, stride: int = 1, padding: int = 0) -> np.ndarray:
    """fp64 direct convolution, left-deep in ``(c, ky, kx)`` order (``dag.py:274-284``).

    ``x``: ``[N, C, H, W]``; ``w``: ``[K, C, R, S]``; returns ``[N, K, P, Q]``.
    """
    xp = pad_input(x, padding)
    w = np.asarray(w, dtype=np.float64)
    n, c_in, h_in, w_in = xp.shape
    k, c_w, kh, kw = w.shape
    assert c_w == c_in, "channel mismatch"
    p = (h_in - kh) // stride + 1
    q = (w_in - kw) // stride + 1
    acc = np.zeros((n, k, p, q), dtype=np.float64)
    for c in range(c_in):
        for ky in range(kh):
            for kx in range(kw):
                win = xp[:, c, ky:ky + stride * (p - 1) + 1:stride,
                         kx:kx + stride * (q - 1) + 1:stride]
                acc += win[:, None, :, :] * w[None, :, c, ky, kx, None, None]
    return acc


def tile_patches(xp: np.ndarray, e: int, m: int, ty: int, tx: int) -> np.ndarray:
    """The m x m input patch of every e x e output tile, ``[n, c, ty, tx, m, m]``:
    tile (ty, tx) reads ``xp[b, c, ty*e + dy, tx*e + dx]`` for ``dy, dx < m``
    (``dag.py:358-363``; pinned to the reference DAG by tests/test_dag_parity.py)."""
    n, c_in = xp.shape[:2]
    patches = np.empty((n, c_in, ty, tx, m, m), dtype=xp.dtype)
    for i in range(ty):
        for j in range(tx):
            patches[:, :, i, j] = xp[:, :, i * e:i * e + m, j * e:j * e + m]
    return patches


def winograd_conv(x: np.ndarray, w: np.ndarray, e: int, padding: int = 0) -> np.ndarray:
    """fp64 Winograd F(e x e, r x r) following the four DAG steps (``dag.py:358-401``)."""
    xp = pad_input(x, padding)
    w = np.asarray(w, dtype=np.float64)
    n, c_in, h_in, w_in = xp.shape
    k, _, r, r2 = w.shape
    assert r == r2, "Winograd needs a square kernel"
    m = e + r - 1
    p_out, q_out = h_in - r + 1, w_in - r + 1
    ty, tx = -(-p_out // e), -(-q_out // e)
    # pad the input so the output domain is a multiple of e (dag.py:291-299)
    need_h, need_w = ty * e + r - 1, tx * e + r - 1
    xp = np.pad(xp, ((0, 0), (0, 0), (0, need_h - h_in), (0, need_w - w_in)))
    mats = winograd_mats.matrices_float(e, r)
    at, g, bt = mats["AT"], mats["G"], mats["BT"]
    # step 1: input transform per (b, c, tile) and kernel transform per (oc, c)
    patches = tile_patches(xp, e, m, ty, tx)
    v = np.einsum("ij,bcyxjk,lk->bcyxil", bt, patches, bt)
    u = np.einsum("ij,ocjk,lk->ocil", g, w, g)
    # steps 2+3: element-wise products summed left-deep over channels
    acc = np.zeros((n, k, ty, tx, m, m))
    for c in range(c_in):
        acc += u[None, :, c, None, None, :, :] * v[:, None, c]
    # step 4: output transform and crop
    y = np.einsum("ij,bkyxjl,ml->bkyxim", at, acc, at)
    y = y.transpose(0, 1, 2, 4, 3, 5).reshape(n, k, ty * e, tx * e)
    return y[:, :, :p_out, :q_out]


def rel_err(y: np.ndarray, ref: np.ndarray) -> float:
    """Norm-wise max error ``||y - ref||_inf / ||ref||_inf``."""
    ref = np.asarray(ref, dtype=np.float64)
    denom = float(np.max(np.abs(ref))) or 1.0
    return float(np.max(np.abs(np.asarray(y, dtype=np.float64) - ref))) / denom


# ---------------------------------------------------------------------------
# the C restatement (oracle/conv_oracle.c), multi-threaded, for big sizes
# ---------------------------------------------------------------------------

_lib = None


def load_c_oracle():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle`")
        lib = ctypes.CDLL(LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        i = ctypes.c_int
        lib.oracle_direct_conv_f32in.argtypes = [fp, fp, dp, i, i, i, i, i, i, i, i, i, i]
        lib.oracle_direct_conv_f32in.restype = i
        lib.oracle_winograd_conv_f32in.argtypes = [fp, fp, dp, i, i, i, i, i, i, i, i,
                                                   dp, dp, dp]
        lib.oracle_winograd_conv_f32in.restype = i
        lib.oracle_set_threads.argtypes = [i]
        lib.oracle_set_threads.restype = i
        _lib = lib
    return _lib


def _fptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def c_direct_conv(x: np.ndarray, w: np.ndarray, stride: int = 1, padding: int = 0,
                  threads: int = 0, images: int | None = None) -> np.ndarray:
    """C oracle, fp32 inputs, fp64 accumulation, same ``(c, ky, kx)`` order.

    ``images`` limits the work to the first ``images`` images (bounded CPU
    baseline samples); the remaining output rows are left zero.
    """
    lib = load_c_oracle()
    lib.oracle_set_threads(threads)
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    n, c, h, wd = x.shape
    k, _, kh, kw = w.shape
    p = (h + 2 * padding - kh) // stride + 1
    q = (wd + 2 * padding - kw) // stride + 1
    y = np.zeros((n, k, p, q), dtype=np.float64)
    nimg = n if images is None else min(images, n)
    rc = lib.oracle_direct_conv_f32in(_fptr(x, ctypes.c_float), _fptr(w, ctypes.c_float),
                                      _fptr(y, ctypes.c_double), nimg, c, h, wd, k, kh, kw,
                                      stride, padding, 0)
    if rc != 0:
        raise ValueError(f"oracle_direct_conv rc={rc}")
    return y


def c_winograd_conv(x: np.ndarray, w: np.ndarray, e: int, padding: int = 0,
                    threads: int = 0, images: int | None = None) -> np.ndarray:
    lib = load_c_oracle()
    lib.oracle_set_threads(threads)
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    n, c, h, wd = x.shape
    k, _, r, _ = w.shape
    mats = winograd_mats.matrices_float(e, r)
    at = np.ascontiguousarray(mats["AT"])
    g = np.ascontiguousarray(mats["G"])
    bt = np.ascontiguousarray(mats["BT"])
    p = h + 2 * padding - r + 1
    q = wd + 2 * padding - r + 1
    y = np.zeros((n, k, p, q), dtype=np.float64)
    nimg = n if images is None else min(images, n)
    rc = lib.oracle_winograd_conv_f32in(_fptr(x, ctypes.c_float), _fptr(w, ctypes.c_float),
                                        _fptr(y, ctypes.c_double), nimg, c, h, wd, k, r, e,
                                        padding, _fptr(at, ctypes.c_double),
                                        _fptr(g, ctypes.c_double), _fptr(bt, ctypes.c_double))
    if rc != 0:
        raise ValueError(f"oracle_winograd_conv rc={rc}")
    return y
