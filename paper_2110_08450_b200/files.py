"""The reference's binary graph / feature / label files, loaded straight into HBM
(formats of graph.py:194-249).

    load_csr_device(path)        MFGC -> DeviceGraph (indptr int64, indices int32)
    load_features_device(path)   FEAT -> [rows, cols] view of a 16-byte-pitched table
    load_labels_device(path)     LABL -> (int64 [rows] tensor, num_classes)
    load_device_graph(csr, feat=None, labels=None) -> DeviceGraph with all three

Payloads stream file -> pinned staging -> HBM through the C-ABI
(sal_load_csr / sal_load_features / sal_load_labels), several host threads
reading chunk k+1 while chunk k is copied; no full host copy is ever made.
Errors are the reference's: BadMagicError, VersionMismatchError and
TruncatedFileError (FormatError subclasses, same messages as
graph.py:176-191), and ValueError from the validation of graph.py:58-65 /
96-100, run on the device.  save_csr / save_features / save_labels write the
same bytes as the reference's writers (graph.py:194-240).
"""

from __future__ import annotations

import ctypes
import os
import struct

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph, DeviceGraph, FeatureMatrix, LabelVector, _pad_cols

CSR_MAGIC, FEAT_MAGIC, LABL_MAGIC = b"MFGC", b"FEAT", b"LABL"
FORMAT_VERSION = 1
DTYPE_F16, DTYPE_F32 = 1, 2

STAGING_BYTES = 256 << 20      # two 128 MB halves
READ_THREADS = max(1, min(16, os.cpu_count() or 1))


class FormatError(Exception):
    """Base class for binary-format problems (graph.py:23-24)."""


class BadMagicError(FormatError):
    pass


class VersionMismatchError(FormatError):
    pass


class TruncatedFileError(FormatError):
    pass


_MAGIC = {_lib.SAL_FILE_CSR: CSR_MAGIC, _lib.SAL_FILE_FEAT: FEAT_MAGIC,
          _lib.SAL_FILE_LABL: LABL_MAGIC}


def read_header(path, kind: int) -> _lib.SalFileHeader:
    """Parse and size-check a file header (host only; raises the reference's errors)."""
    h = _lib.SalFileHeader()
    rc = _lib.lib().sal_file_header_read(os.fsencode(path), kind, ctypes.byref(h))
    if rc == 0:
        return h
    msg = _lib.lib().sal_last_error().decode(errors="replace")
    if rc == _lib.SAL_EBADMAGIC:
        raise BadMagicError(f"bad magic {bytes(h.magic)!r}, expected {_MAGIC[kind]!r}")
    if rc == _lib.SAL_EVERSION:
        raise VersionMismatchError(f"unsupported version {h.version}")
    if rc == _lib.SAL_ETRUNC:
        raise TruncatedFileError(msg)
    if rc == _lib.SAL_EIO:
        raise OSError(msg)
    raise _lib.SalError(f"file header ({rc}): {msg}")


class _Staging:
    """Pinned staging buffer shared by the loaders (allocated on first use)."""
    buf = None

    @classmethod
    def get(cls):
        if cls.buf is None:
            cls.buf = torch.empty(STAGING_BYTES, dtype=torch.uint8).pin_memory()
        return cls.buf


def _run(fn, *args, what: str) -> None:
    rc = fn(*args)
    if rc == _lib.SAL_ETRUNC:
        raise TruncatedFileError(_lib.lib().sal_last_error().decode(errors="replace"))
    if rc == _lib.SAL_EIO:
        raise OSError(_lib.lib().sal_last_error().decode(errors="replace"))
    _lib.check(rc, what)


def load_csr_device(path, device=None, validate: bool = True) -> DeviceGraph:
    """load_csr (graph.py:202-214) into HBM: indptr int64 [n+1], indices int32 [E]."""
    _lib.require_cuda()
    L = _lib.lib()
    h = read_header(path, _lib.SAL_FILE_CSR)
    n, e = int(h.rows), int(h.cols)
    if n >= 2**31 - 1:
        raise ValueError("device graphs are limited to 2^31-1 nodes")
    dev = torch.device(device or "cuda")
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(max(e, 1), dtype=torch.int32, device=dev)[:e]
    st = torch.cuda.current_stream(dev)
    pin = _Staging.get()
    _run(L.sal_load_csr, os.fsencode(path), ctypes.byref(h), indptr.data_ptr(),
         indices.data_ptr() if e else None, pin.data_ptr(), pin.numel(), READ_THREADS,
         _lib.stream_ptr(st), what="load_csr")
    if validate:
        flags = torch.zeros(3, dtype=torch.int32, device=dev)
        _lib.check(L.sal_validate_csr(indptr.data_ptr(), indices.data_ptr() if e else None, n, e,
                                      flags.data_ptr(), _lib.stream_ptr(st)), "validate_csr")
        bad = flags.tolist()
        # CsrGraph.validate order and messages (graph.py:58-65)
        if bad[0]:
            raise ValueError("indptr endpoints inconsistent with edge count")
        if bad[1]:
            raise ValueError("indptr must be non-decreasing")
        if bad[2]:
            raise ValueError("neighbor ID out of range")
    return DeviceGraph(n, indptr, indices)


def load_features_device(path, device=None) -> torch.Tensor:
    """load_features (graph.py:224-232) into HBM: the [rows, cols] view of a
    table whose row pitch is padded to 16 bytes (the gather kernels' layout);
    f16 stays f16, any other dtype code is f32."""
    _lib.require_cuda()
    h = read_header(path, _lib.SAL_FILE_FEAT)
    rows, cols = int(h.rows), int(h.cols)
    dt = torch.float16 if h.dtype == _lib.SAL_F16 else torch.float32
    pad = _pad_cols(cols, h.elem_bytes)
    dev = torch.device(device or "cuda")
    t = torch.empty((rows, pad), dtype=dt, device=dev)
    if pad != cols:
        t[:, cols:].zero_()
    pin = _Staging.get()
    scratch = (torch.empty(pin.numel() // 2, dtype=torch.uint8, device=dev) if pad != cols
               else None)
    _run(_lib.lib().sal_load_features, os.fsencode(path), ctypes.byref(h), t.data_ptr(),
         t.stride(0) * t.element_size(), _lib.ptr(scratch), pin.data_ptr(), pin.numel(),
         READ_THREADS,
         _lib.stream_ptr(torch.cuda.current_stream(dev)), what="load_features")
    return t[:, :cols]


def load_labels_device(path, device=None, validate: bool = True) -> tuple[torch.Tensor, int]:
    """load_labels (graph.py:243-249) into HBM: (int64 [rows], num_classes)."""
    _lib.require_cuda()
    L = _lib.lib()
    h = read_header(path, _lib.SAL_FILE_LABL)
    rows, nc = int(h.rows), int(h.cols)
    dev = torch.device(device or "cuda")
    y = torch.empty(max(rows, 1), dtype=torch.int64, device=dev)[:rows]
    pin = _Staging.get()
    scratch = torch.empty(pin.numel() // 2, dtype=torch.uint8, device=dev)
    st = _lib.stream_ptr(torch.cuda.current_stream(dev))
    _run(L.sal_load_labels, os.fsencode(path), ctypes.byref(h), y.data_ptr(), scratch.data_ptr(),
         pin.data_ptr(), pin.numel(), READ_THREADS, st, what="load_labels")
    if validate and rows:
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(L.sal_validate_labels(y.data_ptr(), rows, nc, flags.data_ptr(), st),
                   "validate_labels")
        if flags.item():
            raise ValueError("label out of range")
    return y, nc


def load_device_graph(csr_path, feat_path=None, labels_path=None, device=None) -> DeviceGraph:
    """One HBM replica from the reference's three files."""
    dg = load_csr_device(csr_path, device)
    if feat_path is not None:
        x = load_features_device(feat_path, device)
        if x.shape[0] != dg.num_nodes:
            raise ValueError(f"feature rows {x.shape[0]} != num_nodes {dg.num_nodes}")
        dg.features = x.as_strided((x.shape[0], x.stride(0)), (x.stride(0), 1))
        dg.num_features = x.shape[1]
    if labels_path is not None:
        y, nc = load_labels_device(labels_path, device)
        if y.shape[0] != dg.num_nodes:
            raise ValueError(f"label rows {y.shape[0]} != num_nodes {dg.num_nodes}")
        dg.labels, dg.num_classes = y, nc
    return dg


# ---------------------------------------------------------------- writers
def save_csr(g: CsrGraph, path) -> None:
    """Same bytes as graph.py:194-199."""
    with open(path, "wb") as f:
        f.write(CSR_MAGIC)
        f.write(struct.pack("<IQQ", FORMAT_VERSION, g.num_nodes, len(g.indices)))
        f.write(np.asarray(g.indptr).astype("<u8").tobytes())
        f.write(np.asarray(g.indices).astype("<u4").tobytes())


def save_features(fm: FeatureMatrix, path) -> None:
    """Same bytes as graph.py:217-221."""
    with open(path, "wb") as f:
        f.write(FEAT_MAGIC)
        f.write(struct.pack("<IQIB3x", FORMAT_VERSION, fm.rows, fm.cols, fm.dtype_code))
        f.write(np.ascontiguousarray(fm.data).tobytes())


def save_labels(y: LabelVector, path) -> None:
    """Same bytes as graph.py:235-239."""
    with open(path, "wb") as f:
        f.write(LABL_MAGIC)
        f.write(struct.pack("<IQI", FORMAT_VERSION, len(y.values), y.num_classes))
        f.write(np.asarray(y.values).astype("<u4").tobytes())


# The reference's loader names (graph.py:202-260).  They return the HBM-resident
# objects every entry point of this package accepts (DeviceGraph, device feature
# rows, (labels, num_classes)), with the reference's header checks and errors.
load_csr = load_csr_device
load_features = load_features_device
load_labels = load_labels_device
