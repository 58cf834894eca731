"""RSPL decomposed-layer files (reference layer.cpp:243-301).

Fixtures under tests/golden/rspl/ were written by the reference's own
write_decomposed_layer (tests/golden/make_rspl_golden.py); rspl.npz holds
what the reference's read_decomposed_layer and forward return for them.
"""
import os

import numpy as np
import pytest

import paper_2504_19449_b200 as rsp

HERE = os.path.dirname(os.path.abspath(__file__))
DIR = os.path.join(HERE, "golden", "rspl")


@pytest.fixture(scope="module")
def rg():
    return np.load(os.path.join(HERE, "golden", "rspl.npz"), allow_pickle=False)


def _path(name):
    return os.path.join(DIR, f"{name}.rspl")


def test_host_reader_matches_reference_reader(rg):
    for name in [str(s) for s in rg["names"]]:
        d = rsp.read_rspl(_path(name))
        s, r = rg[f"{name}.plan"]
        assert d["keep_fraction"] == s and d["rank"] == int(r)
        assert d["kept_width"] == int(np.ceil(s * d["m_in"]))
        # the reference widens the stored f32 to double: identical values
        assert np.array_equal(d["w_cols"].astype(np.float64), rg[f"{name}.w_cols"])
        assert np.array_equal(d["a_r"].astype(np.float64), rg[f"{name}.a_r"])
        assert np.array_equal(d["b_r"].astype(np.float64), rg[f"{name}.b_r"])
        assert np.array_equal(d["comps"].astype(np.int64), rg[f"{name}.comps"])


@pytest.mark.parametrize("name,msg", [
    ("bad_magic", "bad magic"), ("bad_version", "unsupported RSPL version 2"),
    ("truncated_header", "truncated file"), ("truncated_body", "truncated file"),
    ("truncated_plan", "truncated file"), ("bad_rank_field", "inconsistent rank fields"),
])
def test_malformed_files_raise_io_error(rg, name, msg):
    assert name in [str(s) for s in rg["bad_names"]]
    with pytest.raises(rsp.IoError, match=msg):
        rsp.read_rspl(_path(name))


def test_missing_file_is_io_error():
    with pytest.raises(rsp.IoError, match="cannot open layer file"):
        rsp.read_rspl_header(os.path.join(DIR, "does_not_exist.rspl"))


@pytest.mark.gpu
def test_load_forward_save_round_trip(rg, coracle, cuda, tmp_path):
    import torch
    for name in [str(s) for s in rg["names"]]:
        layer = rsp.read_decomposed_layer(_path(name), weight_dtype="f32")
        assert layer.selected_components == [int(c) for c in rg[f"{name}.comps"]]
        s = float(rg[f"{name}.plan"][0])
        for x, y_ref in zip(rg[f"{name}.x"], rg[f"{name}.y"]):
            xt = torch.as_tensor(x.astype(np.float32), device=cuda)
            y = layer.forward(xt).cpu().numpy().astype(np.float64)
            xs = xt.double().cpu().numpy()
            yo, kept = coracle.forward(rg[f"{name}.w_cols"], rg[f"{name}.a_r"], rg[f"{name}.b_r"], s, xs,
                                       return_kept=True)
            assert np.array_equal(layer.selected(xt), kept)
            den = max(np.max(np.abs(yo)), 1e-300)
            assert np.max(np.abs(y - yo)) / den <= 1e-5
            if np.array_equal(xs, x):
                assert np.max(np.abs(y - y_ref)) / max(np.max(np.abs(y_ref)), 1e-300) <= 1e-5
        out = str(tmp_path / f"{name}.rspl")
        rsp.write_decomposed_layer(layer, out)
        assert open(out, "rb").read() == open(_path(name), "rb").read()  # f32: bit-identical file
        bf = rsp.read_decomposed_layer(_path(name), weight_dtype="bf16")
        assert bf.k == layer.k
    sh = rsp.read_decomposed_layer(_path("l48x96"), shard_rank=1, shard_count=2)
    with pytest.raises(rsp.UsageError):
        sh.save_rspl(str(tmp_path / "shard.rspl"))
