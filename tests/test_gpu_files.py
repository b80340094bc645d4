"""f2 loaders into HBM against the arrays the reference's loaders return for
files its writers produced (tests/golden/files.npz), including the semantic
validation errors, multi-chunk streaming and an MFG sampled from a loaded
graph."""
import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden
from paper_2110_08450_b200 import (DeviceGraph, FanoutSpec, SeedBatch, generate_features,
                                   generate_labels, multihop_mfg, synth_graph)
from paper_2110_08450_b200 import files as F

pytestmark = pytest.mark.gpu
FILES = GOLDEN / "files"


def test_load_golden_files_bit_exact():
    z = golden("files")
    dg = F.load_device_graph(FILES / "g.mfgc", FILES / "x16.feat", FILES / "y.labl")
    assert dg.num_nodes == int(z["num_nodes"])
    assert np.array_equal(dg.indptr.cpu().numpy(), z["indptr"])
    assert np.array_equal(dg.indices.cpu().numpy().astype(np.int64), z["indices"])
    x = dg.feature_view()
    assert x.dtype == torch.float16 and x.stride(0) % 8 == 0
    assert np.array_equal(x.cpu().numpy().view(np.uint16), z["x16"].view(np.uint16))
    assert np.array_equal(dg.labels.cpu().numpy(), z["y"]) and dg.num_classes == int(z["num_classes"])
    x32 = F.load_features_device(FILES / "x32.feat")
    assert x32.dtype == torch.float32 and x32.stride(0) == 8
    assert np.array_equal(x32.cpu().numpy().view(np.uint32), z["x32"].view(np.uint32))


def test_semantic_errors_match_reference():
    z = golden("files")
    loaders = {"g.mfgc": F.load_csr_device, "y.labl": F.load_labels_device}
    seen = 0
    for name, tag, cls, msg in z["errors"]:
        if tag not in ("badindex", "decreasing", "endpoint", "start", "badlabel"):
            continue
        with pytest.raises(ValueError) as ei:
            loaders[name](FILES / f"{tag}_{name}")
        assert cls == "ValueError" and str(ei.value) == msg, (tag, str(ei.value), msg)
        seen += 1
    assert seen == 5


def test_multi_chunk_streaming(tmp_path, monkeypatch):
    """A staging buffer much smaller than the payload: many chunks, odd row
    sizes (f = 37 fp16 -> 74 B rows, pitch 80 B), labels widened per chunk."""
    g = synth_graph(20000, 12, 3.0, seed=2)
    fm = generate_features(20000, 37, "f16", seed=2)
    y = generate_labels(20000, 50, seed=2)
    F.save_csr(g, tmp_path / "g.mfgc")
    F.save_features(fm, tmp_path / "x.feat")
    F.save_labels(y, tmp_path / "y.labl")
    monkeypatch.setattr(F._Staging, "buf", torch.empty(3 * 4096 * 2 + 100,
                                                       dtype=torch.uint8).pin_memory())
    monkeypatch.setattr(F, "READ_THREADS", 3)
    dg = F.load_device_graph(tmp_path / "g.mfgc", tmp_path / "x.feat", tmp_path / "y.labl")
    assert np.array_equal(dg.indptr.cpu().numpy(), g.indptr)
    assert np.array_equal(dg.indices.cpu().numpy(), g.indices)
    assert np.array_equal(dg.feature_view().cpu().numpy().view(np.uint16), fm.data.view(np.uint16))
    assert np.array_equal(dg.labels.cpu().numpy(), y.values)
    # an MFG from the loaded replica equals one from the uploaded host graph
    seeds = SeedBatch(3, np.arange(0, 20000, 37)[:256])
    a = multihop_mfg(dg, seeds, FanoutSpec((15, 10, 5)), 1).digest()
    b = multihop_mfg(DeviceGraph.from_host(g), seeds, FanoutSpec((15, 10, 5)), 1).digest()
    assert a == b
