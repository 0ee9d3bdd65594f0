"""Host-side logic of the experiment runner (CPU): configuration validation,
cell formatting, CSV/JSON rendering and argument parsing mirror the
reference CLI (cli.py:39-330)."""

import csv
import io
import json

import pytest

from paper_2602_05191_b200 import cli


def test_run_config_validation():
    spec = cli.WorkloadSpec(context_len=256, head_dim=16)
    with pytest.raises(ValueError, match="unknown method"):
        cli.RunConfig(workload=spec, input_path=None, method="nope")
    with pytest.raises(ValueError, match="exactly one"):
        cli.RunConfig(workload=spec, input_path="x.dpkv", method="full")
    with pytest.raises(ValueError, match="exactly one"):
        cli.RunConfig(workload=None, input_path=None, method="full")
    with pytest.raises(ValueError, match="must exceed sink"):
        cli.WorkloadSpec(context_len=60, head_dim=16)


def test_record_validation():
    base = dict(layer=0, head=0, step=0, method="full", p1=None, p2=None, k=None, m=None, B=None,
                clusters_total=None, clusters_selected=None, clusters_exact=None, exact_tokens=3, est_mass=None,
                recovered_mass=1.0, violation=False, rel_err=0.0)
    cli.ExperimentRecord(**base)
    with pytest.raises(ValueError, match="recovered_mass out of range"):
        cli.ExperimentRecord(**dict(base, recovered_mass=1.1))
    with pytest.raises(ValueError, match="rel_err"):
        cli.ExperimentRecord(**dict(base, rel_err=-1.0))


def test_csv_and_json_rendering():
    rows = [{"a": 1, "b": None, "c": True, "d": 0.1234567890123456, "e": "x"}]
    cols = ["a", "b", "c", "d", "e"]
    text = cli.render(rows, cols, "csv")
    assert text == "a,b,c,d,e\n1,,1,0.123456789012,x\n"
    j = json.loads(cli.render(rows, cols, "json"))
    assert j == [{"a": 1, "b": None, "c": True, "d": 0.1234567890123456, "e": "x"}]
    assert list(csv.reader(io.StringIO(text)))[0] == cols


def test_parser_mirrors_reference_flags():
    p = cli.build_parser()
    a = p.parse_args(["run", "--n", "256", "--d", "16", "--method", "doublep", "--preset", "qwen-default",
                      "--p2", "0.5"])
    assert cli._thresholds(a) == (0.99, 0.5)
    assert a.window == 64 and a.sink == 4 and a.tokens_per_cluster == 32 and a.target_p == 0.95
    s = p.parse_args(["sweep", "--n", "256", "--d", "16", "--methods", "doublep,token_topk", "--k-grid", "4,8"])
    assert s.k_grid == "4,8" and s.methods == "doublep,token_topk"
    f = p.parse_args(["figs", "--table", "tracking", "--n", "256", "--d", "16"])
    assert f.k_list == "64,256,1024"
    assert cli.CSV_COLUMNS[-1] == "rel_err" and len(cli.CSV_COLUMNS) == 17


def test_atomic_emit(tmp_path):
    out = tmp_path / "o.csv"
    cli.emit("x\n", str(out))
    assert out.read_text() == "x\n"
    assert [p.name for p in tmp_path.iterdir()] == ["o.csv"]
