"""f2 file formats on the host: header parsing and its errors against the
reference's own behaviour on malformed files (tests/golden/files.npz records
the exception class + message the reference loaders raised), and the writers
against files written by the reference's writers."""
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_2110_08450_b200 import files as F
from paper_2110_08450_b200 import _lib
from paper_2110_08450_b200.graph import CsrGraph, FeatureMatrix, LabelVector

FILES = GOLDEN / "files"
KIND = {"g.mfgc": _lib.SAL_FILE_CSR, "x16.feat": _lib.SAL_FILE_FEAT, "y.labl": _lib.SAL_FILE_LABL}


def _variant(good: bytes, tag: str) -> bytes:
    if tag == "badmagic":
        return b"XXXX" + good[4:]
    if tag == "badversion":
        return good[:4] + (2).to_bytes(4, "little") + good[8:]
    assert tag.startswith("trunc")
    return good[:int(tag[5:])]


def test_header_errors_match_reference(tmp_path):
    z = golden("files")
    seen = 0
    for name, tag, cls, msg in z["errors"]:
        if tag not in ("badmagic", "badversion") and not tag.startswith("trunc"):
            continue  # semantic faults are checked on the device (test_gpu_files)
        p = tmp_path / f"{tag}_{name}"
        p.write_bytes(_variant((FILES / name).read_bytes(), tag))
        with pytest.raises(getattr(F, cls)) as ei:
            F.read_header(p, KIND[name])
        assert str(ei.value) == msg, (name, tag)
        assert isinstance(ei.value, F.FormatError)
        seen += 1
    assert seen == 21


def test_headers_of_good_files():
    z = golden("files")
    h = F.read_header(FILES / "g.mfgc", _lib.SAL_FILE_CSR)
    assert (h.rows, h.cols, h.payload_offset) == (int(z["num_nodes"]), len(z["indices"]), 24)
    h = F.read_header(FILES / "x16.feat", _lib.SAL_FILE_FEAT)
    assert (h.rows, h.cols, h.dtype, h.elem_bytes) == (700, 20, _lib.SAL_F16, 2)
    h = F.read_header(FILES / "x32.feat", _lib.SAL_FILE_FEAT)
    assert (h.rows, h.cols, h.dtype, h.elem_bytes) == (700, 7, _lib.SAL_F32, 4)
    h = F.read_header(FILES / "y.labl", _lib.SAL_FILE_LABL)
    assert (h.rows, h.cols, h.payload_offset) == (700, int(z["num_classes"]), 20)
    with pytest.raises(OSError):
        F.read_header(FILES / "missing.mfgc", _lib.SAL_FILE_CSR)


def test_writers_reproduce_reference_bytes(tmp_path):
    z = golden("files")
    g = CsrGraph(int(z["num_nodes"]), z["indptr"], z["indices"])
    F.save_csr(g, tmp_path / "g.mfgc")
    F.save_features(FeatureMatrix(700, 20, z["x16"]), tmp_path / "x16.feat")
    F.save_features(FeatureMatrix(700, 7, z["x32"]), tmp_path / "x32.feat")
    F.save_labels(LabelVector(z["y"], int(z["num_classes"])), tmp_path / "y.labl")
    for name in ("g.mfgc", "x16.feat", "x32.feat", "y.labl"):
        assert (tmp_path / name).read_bytes() == (FILES / name).read_bytes(), name
