"""`python -m paper_2604_02715_b200 run|verify|calibrate` on the GPU (reference cli.py:92-208)."""

import json

import pytest

pytestmark = pytest.mark.gpu


def test_cli_run_passes_and_reports(capsys, tmp_path):
    from paper_2604_02715_b200.__main__ import main

    out = tmp_path / "r.json"
    assert main(["run", "--model", "4,8,64,128", "--iterations", "2", "--tokens", "8", "--seeds", "2",
                 "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["passed"] and len(doc["runs"]) == 2
    r = doc["runs"][0]
    assert r["bit_identical"] and r["violations"] == 0 and r["arena_peak_bytes"] == r["expected_peak_bytes"]
    assert main(["run", "--model", "4,8,64,128", "--alpha", "0.5", "--host-codec", "--mode", "sequential"]) == 0


def test_cli_verify_and_container_run(tmp_path):
    from paper_2604_02715_b200.__main__ import main

    xpgw, xpgc = tmp_path / "m.xpgw", tmp_path / "m.xpgc"
    assert main(["generate", str(xpgw), "--model", "3,4,64,128"]) == 0
    assert main(["compress", str(xpgw), str(xpgc)]) == 0
    assert main(["verify", str(xpgw), str(xpgc)]) == 0
    assert main(["run", "--container", str(xpgw), "--iterations", "1"]) == 0


def test_cli_calibrate(capsys):
    from paper_2604_02715_b200.__main__ import main

    assert main(["calibrate", "--model", "4,8,512,1024", "--tokens", "64"]) == 0
    doc = json.loads(capsys.readouterr().out)
    assert doc["b_host"] > 0 and doc["b_dev"] > 0 and doc["tau_comp_theory"] > 0
    assert 0.0 <= doc["knee_alpha"] <= 1.0 and 0.5 < doc["compression_ratio"] < 0.8
