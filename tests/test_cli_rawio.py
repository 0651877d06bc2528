"""CLI + raw tensor format (mirrors the reference's test_cli.py)."""
import json

import numpy as np
import pytest

import paper_2504_11681_b200 as T
from paper_2504_11681_b200.cli import main
from paper_2504_11681_b200.rawio import read_raw_matrix, read_raw_tensor, write_raw_matrix, write_raw_tensor


def test_count_ops_output(capsys):
    assert main(["count-ops", "4", "1"]) == 0
    assert "3 / 8 = 0.375" in capsys.readouterr().out
    assert main(["count-ops", "4", "4"]) == 0
    assert "8 / 8 = 1" in capsys.readouterr().out
    assert main(["count-ops", "256", "64", "256"]) == 0
    assert "1728 / 2048" in capsys.readouterr().out


def test_raw_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(1)
    a = (rng.standard_normal((2, 3, 4, 5)) + 1j * rng.standard_normal((2, 3, 4, 5))).astype(np.complex64)
    p = tmp_path / "a.bin"
    write_raw_tensor(str(p), a)
    assert p.stat().st_size == 16 + a.size * 8
    assert np.array_equal(read_raw_tensor(str(p)), a)
    raw = p.read_bytes()
    assert np.frombuffer(raw[:16], "<u4").tolist() == [2, 3, 4, 5]
    (tmp_path / "t.bin").write_bytes(raw[:-4])
    with pytest.raises(T.FnofuseError):
        read_raw_tensor(str(tmp_path / "t.bin"))
    (tmp_path / "x.bin").write_bytes(raw + b"\0")
    with pytest.raises(T.FnofuseError):
        read_raw_tensor(str(tmp_path / "x.bin"))
    w = T.ComplexMatrix.random(3, 7, rng)
    write_raw_matrix(str(tmp_path / "w.bin"), w)
    assert np.array_equal(read_raw_matrix(str(tmp_path / "w.bin")).values, w.values)


def test_fno_run_config_mismatch_and_io_error(tmp_path, capsys):
    cfg = T.FnoLayerConfig(2, 16, 16, 1, 64, 1, 16, rank=1)
    x = T.random_spectral(cfg, np.random.default_rng(4))
    inp = tmp_path / "in.bin"
    write_raw_tensor(str(inp), x.data)
    conf = tmp_path / "layer.json"
    conf.write_text(json.dumps({"layer": {"batch": 3, "output_dim": 16, "keep_x": 1, "keep_y": 16, "rank": 1}}))
    assert main(["fno-run", "--input", str(inp), "--out", str(tmp_path / "o.bin"), "--config", str(conf)]) == 2
    assert "disagrees" in capsys.readouterr().err
    conf.write_text(json.dumps({"layer": {"output_dim": 16, "keep_x": 1, "keep_y": 16, "rank": 1}}))
    assert main(["fno-run", "--input", str(tmp_path / "nope.bin"), "--out", str(tmp_path / "o.bin"),
                 "--config", str(conf)]) == 3


@pytest.mark.gpu
def test_fno_run_matches_library(tmp_path):
    """test_cli.py:85-111 equivalent on the GPU path."""
    cfg = T.FnoLayerConfig(2, 16, 24, 1, 64, 1, 16, rank=1)
    rng = np.random.default_rng(4)
    x = T.random_spectral(cfg, rng)
    w = T.ComplexMatrix.random(16, 24, rng)
    inp, wf, outp, ledp = (tmp_path / n for n in ("in.bin", "w.bin", "out.bin", "ledger.json"))
    write_raw_tensor(str(inp), x.data)
    write_raw_matrix(str(wf), w)
    conf = tmp_path / "layer.json"
    conf.write_text(json.dumps({"layer": {"output_dim": 24, "keep_x": 1, "keep_y": 16, "rank": 1},
                                "tiles": T.DEFAULT_TILES.to_json_dict()}))
    assert main(["fno-run", "--input", str(inp), "--out", str(outp), "--config", str(conf), "--weights", str(wf),
                 "--mode", "fully_fused", "--ledger-out", str(ledp)]) == 0
    got = read_raw_tensor(str(outp))
    want, led = T.run_layer(cfg, x, w, mode="fully_fused")
    assert np.array_equal(got, want.data)
    doc = json.loads(ledp.read_text())
    assert doc == led.to_json_dict() and doc["kernel_launches"] == 1
