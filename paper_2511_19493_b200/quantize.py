"""QLORA factor quantisation — drop-in for quantize.py (quantize.py:1-140).

``quantize`` runs on the GPU (csrc/quant.cu): per-column absmax/127 INT8
with round-half-even and clip to +-127, f32 / f16 casts, NF4 64-blocks of the
column-major flatten against the 16-level codebook.  ``QuantFactor`` keeps
the reference's fields and decode semantics so downstream code (file
writers, ``entry``) reads it unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

MODES = ("f32", "f16", "i8", "nf4")
BYTES_PER_ELEMENT = {"f32": 4.0, "f16": 2.0, "i8": 1.0, "nf4": 0.5}
NF4_BLOCK = 64
NF4_CODEBOOK = np.array([
    -1.0, -0.6961928009986877, -0.5250730514526367, -0.39491748809814453,
    -0.28444138169288635, -0.18477343022823334, -0.09105003625154495, 0.0,
    0.07958029955625534, 0.16093020141124725, 0.24611230194568634, 0.33791524171829224,
    0.44070982933044434, 0.5626170039176941, 0.7229568362236023, 1.0], dtype=np.float64)


def nf4_max_gap() -> float:
    return float(np.diff(NF4_CODEBOOK).max())


@dataclass
class QuantFactor:
    """Quantised matrix + metadata (quantize.py:49-72)."""

    mode: str
    shape: tuple
    data: np.ndarray
    scales: np.ndarray | None = None

    def dequantize(self) -> np.ndarray:
        return dequantize(self)

    def payload_nbytes(self) -> int:
        total = self.data.nbytes
        if self.scales is not None:
            total += self.scales.nbytes
        return total


def _device_quantize(F, n: int, r: int, mode: str):
    """F: (n, r) f64 device tensor.  Returns (data tensor, scales tensor|None)."""
    import torch
    dev = F.device
    m = _lib.Q_MODES[mode]
    if mode == "i8":
        data = torch.empty((n, r), dtype=torch.int8, device=dev)
        scales = torch.empty(r, dtype=torch.float64, device=dev)
    elif mode == "f32":
        data = torch.empty((n, r), dtype=torch.float32, device=dev)
        scales = None
    elif mode == "f16":
        data = torch.empty((n, r), dtype=torch.float16, device=dev)
        scales = None
    else:
        nb = (n * r + NF4_BLOCK - 1) // NF4_BLOCK
        data = torch.empty(nb * NF4_BLOCK // 2, dtype=torch.uint8, device=dev)
        scales = torch.empty(nb, dtype=torch.float64, device=dev)
    return data, scales, m


def factor_quantize(Q, Wr, mode: str):
    """factor = Q @ Wr on the device, then quantise (proximity.py:403-405).
    Q: (n, k) f64 device; Wr: (k, r) f64 (device tensor or host array).
    Returns device tensors (data, scales)."""
    import torch
    n, k = Q.shape
    r = Wr.shape[1]
    dev = Q.device
    wr = Wr if isinstance(Wr, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(Wr, dtype=np.float64)).to(dev)
    F = torch.empty((n, r), dtype=torch.float64, device=dev)
    parts = torch.empty(_lib.load().rfxc_gram_parts(n) * r, dtype=torch.float64, device=dev)
    data, scales, m = _device_quantize(F, n, r, mode)
    sc = scales if scales is not None else torch.empty(1, dtype=torch.float64, device=dev)
    _lib.call("rfxc_factor_quantize", _lib.ptr(Q), n, k, _lib.ptr(wr), r, m, _lib.ptr(F),
              _lib.ptr(parts), _lib.ptr(sc), _lib.ptr(data), _lib.stream_handle())
    return data, scales


def device_dequantize(data, scales, n: int, r: int, mode: str):
    import torch
    dq = torch.empty((n, r), dtype=torch.float64, device=data.device)
    sc = scales if scales is not None else torch.empty(1, dtype=torch.float64,
                                                       device=data.device)
    _lib.call("rfxc_dequantize", _lib.ptr(data), _lib.ptr(sc), n, r, _lib.Q_MODES[mode],
              _lib.ptr(dq), _lib.stream_handle())
    return dq


def to_host(mode: str, shape, data, scales) -> QuantFactor:
    d = data.cpu().numpy()
    if mode in ("f32", "f16", "i8"):
        d = d.reshape(shape)
    s = None if scales is None else scales.cpu().numpy().astype(np.float64)
    return QuantFactor(mode, tuple(shape), d, s)


def quantize(values, mode: str) -> QuantFactor:
    """Drop-in for quantize.quantize (quantize.py:83-117), on the GPU."""
    import torch
    if mode not in MODES:
        raise ValueError(f"unknown quantization mode {mode!r}; expected one of {MODES}")
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim not in (1, 2):
        raise ValueError("quantize expects a 1-D block or a 2-D matrix")
    if not np.isfinite(arr).all():
        raise ValueError("quantize requires finite inputs")
    shape = arr.shape
    mat = arr.reshape(-1, 1) if arr.ndim == 1 else arr
    dev = _lib.require_cuda()
    n, r = mat.shape
    Q = torch.from_numpy(np.ascontiguousarray(mat)).to(dev)
    data, scales = factor_quantize(Q, np.eye(r), mode)
    return to_host(mode, shape, data, scales)


def dequantize(qf: QuantFactor) -> np.ndarray:
    """Host decode with the reference's semantics (quantize.py:120-140); used
    by entry()/file I/O, not by the device path (which keeps its own copy)."""
    if qf.mode in ("f32", "f16"):
        return qf.data.astype(np.float64)
    if qf.mode == "i8":
        mat = qf.data.astype(np.float64)
        return mat * qf.scales[0] if mat.ndim == 1 else mat * qf.scales[None, :]
    if qf.mode == "nf4":
        n_elem = int(np.prod(qf.shape))
        nb = qf.scales.shape[0]
        codes = np.empty(nb * NF4_BLOCK, dtype=np.uint8)
        codes[0::2] = qf.data & 0x0F
        codes[1::2] = qf.data >> 4
        vals = NF4_CODEBOOK[codes].reshape(nb, NF4_BLOCK) * qf.scales[:, None]
        flat = vals.reshape(-1)[:n_elem]
        return flat if len(qf.shape) == 1 else flat.reshape(qf.shape, order="F")
    raise ValueError(f"unknown quantization mode {qf.mode!r}")
