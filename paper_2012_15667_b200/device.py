"""B200 machine model and the device projection of the reference's model.

The reference's two-level machine ``HwModel(s, s_sm, n_p)``
(``pkg/src/convio/model.py:123-156``) is instantiated for B200 as:

* ``s_sm`` -- fast-memory words per SM = the 64 Ki 32-bit registers (where
  the output-stationary block keeps its ``xyz`` partial sums) plus the
  228 KiB of shared memory (where channel stages are staged):
  ``65536 + 58368 = 123904`` words;
* ``n_p = 296`` -- two resident blocks on each of the 148 SMs, the
  ``s_sm = 2 * (s // n_p)`` convention of the reference model;
* ``s = n_p * s_sm / 2``.

So the Table-1 ``s_b`` axis runs over powers of two up to 32768 words.  A
``TileConfig``'s *device projection* (legality, grid, threads, shared
memory, channels per stage) is computed by the C-ABI's ``convio_query``.
"""

from __future__ import annotations

from .model import HwModel, ConvShape

B200_SMS = 148
B200_REGS_WORDS = 65536
B200_SMEM_WORDS = 228 * 1024 // 4
B200_S_SM = B200_REGS_WORDS + B200_SMEM_WORDS
B200_N_P = 2 * B200_SMS


def b200_hw_model(sms: int = B200_SMS) -> HwModel:
    """The B200 instance of the reference machine model."""
    n_p = 2 * sms
    return HwModel(s=n_p * (B200_S_SM // 2), s_sm=B200_S_SM, n_p=n_p)


def direct_flops(n, c, k, p, q, r, s) -> int:
    """Algorithmic flops of a direct convolution (2 per multiply-add)."""
    return 2 * n * k * c * r * s * p * q


def winograd_gemm_flops(n, c, k, p, q, e, r=3) -> int:
    """Element-wise (batched GEMM) flops of F(e x e, r x r): ``2 m^2 K C tiles``."""
    m = e + r - 1
    tiles = n * (-(-p // e)) * (-(-q // e))
    return 2 * m * m * k * c * tiles


def shape_of(n, c, h, w, k, r, stride, pad) -> ConvShape:
    """The reference ``ConvShape`` of a padded layer (padding as geometry)."""
    p = (h + 2 * pad - r) // stride + 1
    q = (w + 2 * pad - r) // stride + 1
    return ConvShape.from_output(q, p, k, c, r, r, stride, n)


def device_projection(x_shape, w_shape, tile, stride=1, padding=0, layout="CHW",
                      algorithm="direct") -> dict:
    """Launch shape / legality of ``tile`` on this device (``convio_query``)."""
    from .conv import query
    return query(x_shape, w_shape, stride, padding, layout, tile, algorithm)
