"""The "b200" kernel backend: the reference plugin interface of
``certkv._kernels`` (NAME, block_logmass, fused_attend; pure.py:13-66)
served by the CUDA library.  Parity surface only: per-call host arrays make
it transfer-bound, the hot path never goes through it.
"""

import ctypes

import numpy as np
import torch

from . import _lib

NAME = "b200"


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the b200 kernel backend needs a CUDA device")
    return torch.device("cuda")


def _s():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def block_logmass(scores, bounds):
    """Per-block (max, exp-sum, log-mass) in float64 (pure.py:16-36)."""
    lib = _lib.load()
    s = torch.as_tensor(np.ascontiguousarray(scores, dtype=np.float64), device=_dev())
    b = torch.as_tensor(np.ascontiguousarray(bounds, dtype=np.int64), device=_dev())
    nb = int(b.shape[0]) - 1
    if nb <= 0:
        e = np.empty(0, dtype=np.float64)
        return e, e.copy(), e.copy()
    out = torch.empty((3, nb), dtype=torch.float64, device=_dev())
    _lib.check(lib.ckv_block_logmass(s.data_ptr(), b.data_ptr(), nb, out[0].data_ptr(),
                                     out[1].data_ptr(), out[2].data_ptr(), _s()),
               "ckv_block_logmass")
    o = out.cpu().numpy()
    return o[0].copy(), o[1].copy(), o[2].copy()


def fused_attend(scores, values, bounds):
    """Single-pass online-softmax attend with float32 state (pure.py:39-66)."""
    lib = _lib.load()
    s = torch.as_tensor(np.ascontiguousarray(scores, dtype=np.float32), device=_dev())
    v = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float32), device=_dev())
    b = torch.as_tensor(np.ascontiguousarray(bounds, dtype=np.int64), device=_dev())
    nb, d = int(b.shape[0]) - 1, int(v.shape[1])
    out = torch.empty(d, dtype=torch.float32, device=_dev())
    ml = torch.empty(2, dtype=torch.float32, device=_dev())
    _lib.check(lib.ckv_fused_attend(s.data_ptr(), v.data_ptr(), b.data_ptr(), nb, d,
                                    out.data_ptr(), ml.data_ptr(), _s()), "ckv_fused_attend")
    m = ml.cpu().numpy()
    return out.cpu().numpy(), np.float32(m[0]), np.float32(m[1])
