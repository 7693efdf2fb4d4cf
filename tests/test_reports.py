"""The reference-schema benchmark reports with GPU columns (scripts/refbench,
SURVEY 8f rank 4): the committed reports of a GPU run parse as CSV / JSON, keep
the reference's columns and keys first (bench.cpp:356-430), carry the GPU
columns, and are read back by the reference's own parsers
(cfar_report_from_csv / _json, bench.cpp:446-528) through `refbench parse`."""
import csv
import io
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPORTS = os.path.join(ROOT, "profiles", "r02_reports")
PARSER = os.path.join(ROOT, "scripts", "refbench", "_build", "refbench_reference")

CFAR_REF_COLS = ["guard", "background", "naive_mean_s", "naive_std_s", "ii_mean_s", "ii_std_s", "ratio"]
PIPE_REF_COLS = ["step", "ca_mean_s", "ca_std_s", "ii_mean_s", "ii_std_s"]


def _read(name):
    with open(os.path.join(REPORTS, name)) as f:
        return f.read()


def test_cfar_csv_has_reference_columns_then_gpu_columns():
    rows = list(csv.reader(io.StringIO(_read("cfar_b200.csv"))))
    assert rows[0][:7] == CFAR_REF_COLS
    assert rows[0][7:] == ["dev_naive_s", "dev_ii_s", "dev_ratio", "dev_ii_hbm_frac"]
    grid = [(int(r[0]), int(r[1])) for r in rows[1:]]
    assert grid == [(4, 8), (4, 12), (8, 8), (8, 12)]  # bench.hpp:18
    for r in rows[1:]:
        naive, ii, ratio = float(r[7]), float(r[8]), float(r[9])
        assert naive > 0 and ii > 0 and abs(ratio - naive / ii) < 1e-6 * ratio
        assert 0 < float(r[10]) < 1


def test_cfar_json_keeps_reference_keys():
    j = json.loads(_read("cfar_b200.json"))
    assert j["mode"] == "cfar" and len(j["rows"]) == 4
    for row in j["rows"]:
        for k in ["guard", "background", "naive_mean_s", "naive_std_s", "ii_mean_s", "ii_std_s", "ratio"]:
            assert k in row
        assert row["e2e_ii_s"] == row["ii_mean_s"]
        assert row["dev_ii_s"] > 0 and row["dev_naive_s"] > 0
    assert "gpu_note" in j


def test_pipeline_reports_gpu_rows():
    rows = list(csv.reader(io.StringIO(_read("pipeline_b200.csv"))))
    assert rows[0][:5] == PIPE_REF_COLS and rows[0][5:] == ["dev_ca_s", "dev_ii_s"]
    names = [r[0] for r in rows[1:]]
    assert names[-1] == "Total" and len(names) == 5
    total = rows[-1]
    assert float(total[5]) > 0 and float(total[6]) > 0
    j = json.loads(_read("pipeline_b200.json"))
    assert j["rows"][0]["dev_ca_s"] is None and j["rows"][4]["dev_ii_s"] > 0
    text = _read("pipeline_b200.text")
    assert "GPU columns" in text and text.startswith("Pipeline step timings")


@pytest.mark.skipif(not os.path.exists(PARSER), reason="refbench not built (needs /root/reference)")
@pytest.mark.parametrize("mode,fmt", [("cfar", "csv"), ("cfar", "json"), ("pipeline", "csv"), ("pipeline", "json")])
def test_reference_parsers_read_the_augmented_reports(mode, fmt):
    out = subprocess.run([PARSER, "parse", mode, fmt, os.path.join(REPORTS, f"{mode}_b200.{fmt}")],
                         capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert len(lines) == (4 if mode == "cfar" else 5)
