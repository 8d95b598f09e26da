"""Block fits for keys (per-channel INT8) and values (per-group INT4), fp64.

Restates ``quantizer.py`` of the reference (see each function).  TEST
INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.
"""

import numpy as np

KEY_LEVELS = 255.0   # quantizer.py:35 (codes -128..127)
VALUE_LEVELS = 15.0  # quantizer.py:36 (codes 0..15)


def pairwise_sum128(row):
    """NumPy's float64 pairwise sum for one contiguous row of <=128 values.

    ``np.sum(x, axis=-1)`` over a contiguous row reduces with 8 running
    accumulators then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); rows shorter
    than 8 are summed left to right.  The reference annotations
    (quantizer.py:214-216) depend on this order, and the CUDA fill kernel
    reproduces it; ``tests/test_oracle_golden.py`` pins it against np.sum.
    """
    a = [float(x) for x in row]
    n = len(a)
    if n < 8:
        acc = 0.0
        for x in a:
            acc += x
        return acc
    r = a[:8]
    i = 8
    stop = n - (n % 8)
    while i < stop:
        for j in range(8):
            r[j] += a[i + j]
        i += 8
    acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        acc += a[i]
        i += 1
    return acc


def _reject_nonfinite(block, what):
    """quantizer.py:98-102: name the first offending channel."""
    if not np.all(np.isfinite(block)):
        where = np.argwhere(~np.isfinite(np.atleast_2d(block)))
        raise ValueError(f"non-finite {what} entry in channel {int(where[0][-1])}")


def _refine(x, step, base, lo_code, hi_code):
    """Round-half-even then one strict +-1 neighbour pass (quantizer.py:118-130).

    The +1 candidate is taken relative to the code *after* the -1 pass, and a
    candidate replaces the current code only when its computed reconstruction
    error is strictly smaller.
    """
    code = np.clip(np.rint((x - base) / step), lo_code, hi_code)
    err = np.abs(x - (code * step + base))
    for delta in (-1.0, 1.0):
        trial = np.clip(code + delta, lo_code, hi_code)
        trial_err = np.abs(x - (trial * step + base))
        take = trial_err < err
        code = np.where(take, trial, code)
        err = np.where(take, trial_err, err)
    return code


def fit_key_block(keys):
    """Per-channel INT8 fit of one (B, d) block -> (codes i8, scale f64, offset f64).

    quantizer.py:133-161 with _fit_affine (105-115): scale=(max-min)/255,
    offset=min+128*scale, constant channels get scale 1 / offset = the constant.
    """
    k = np.asarray(keys, dtype=np.float64)
    if k.ndim != 2:
        raise ValueError(f"expected a 2-D block, got shape {k.shape}")
    _reject_nonfinite(k, "key")
    lo = k.min(axis=0)
    hi = k.max(axis=0)
    flat = hi == lo
    scale = np.where(flat, 1.0, (hi - lo) / KEY_LEVELS)
    offset = np.where(flat, lo, lo + 128.0 * scale)
    codes = _refine(k, scale[None, :], offset[None, :], -128.0, 127.0)
    return codes.astype(np.int8), scale, offset


def fit_value_block(values, group):
    """Per-(token, group) INT4 fit of one (B, d) block.

    quantizer.py:178-194, 220-230: scale=(max-min)/15 (1 if constant),
    offset=min; returns (codes u8 (B,d), scale (B,d/g), offset (B,d/g)).
    """
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 2:
        raise ValueError(f"expected a 2-D block, got shape {v.shape}")
    _reject_nonfinite(v, "value")
    b, d = v.shape
    if group <= 0 or d % group:
        raise ValueError(f"group size {group} does not divide head dim {d}")
    gv = v.reshape(b, d // group, group)
    lo = gv.min(axis=-1)
    hi = gv.max(axis=-1)
    scale = np.where(hi == lo, 1.0, (hi - lo) / VALUE_LEVELS)
    codes = _refine(gv, scale[..., None], lo[..., None], 0.0, 15.0)
    return codes.reshape(b, d).astype(np.uint8), scale, lo


def narrow_key_meta(scale, offset):
    """Device widths for key metadata: FP32 (cache.py:11-13 accounting)."""
    return (np.asarray(scale).astype(np.float32).astype(np.float64),
            np.asarray(offset).astype(np.float32).astype(np.float64))


def narrow_value_meta(scale, offset):
    """Device widths for value metadata: FP16 (cache.py:11-13 accounting)."""
    return (np.asarray(scale).astype(np.float16).astype(np.float64),
            np.asarray(offset).astype(np.float16).astype(np.float64))


def dequant_keys(codes, scale, offset):
    """codes*scale + offset in fp64, two roundings (quantizer.py:164-166)."""
    return codes.astype(np.float64) * scale[..., None, :] + offset[..., None, :]


def dequant_values(codes, scale, offset, group):
    """Per-group affine reconstruction in fp64 (quantizer.py:197-204)."""
    shape = codes.shape
    g = codes.astype(np.float64).reshape(shape[:-1] + (shape[-1] // group, group))
    return (g * scale[..., None] + offset[..., None]).reshape(shape)


def value_annotations(values, recon):
    """(eta, nu): max over tokens of the L2 error / value norm (quantizer.py:207-217).

    Squares, pairwise channel sum (np.sum), sqrt, then max -- the canonical
    order the reference documents at quantizer.py:27-28.
    """
    v = np.asarray(values, dtype=np.float64)
    diff = recon - v
    eta = float(np.sqrt(np.sum(diff * diff, axis=-1)).max())
    nu = float(np.sqrt(np.sum(v * v, axis=-1)).max())
    return eta, nu
