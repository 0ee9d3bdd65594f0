"""pyexport on the B200 path (paper_2602_05191_b200.capture; reference
pkg/pyexport/src/pyexport/{capture,exporter,cli}.py).

CPU: the dumps this package writes for the reference's synthetic-llama are
byte-identical to the ones the reference exporter wrote
(oracle/gen_golden_pyexport.py -> tests/golden/pyexport_synth_*.dpkv), and
the exporter's error contract (test_export.py:154-192) holds.
GPU: a capture taken on the device feeds the clustered cache directly, and
the decode step on that real-model attention passes the SURVEY 8c parity
protocol against the oracle; dense weights from the dump reproduce the
runtime's own probabilities (test_export.py:55-85)."""

import json
import os

import numpy as np
import pytest
import torch

from paper_2602_05191_b200 import capture as C

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PROMPT = ("The export path is exercised with a prompt long enough to give the attention maps some structure: "
          "repeated phrases, punctuation, and a little variation.")
STEPS = 6


@pytest.mark.parametrize("dtype", ["float32", "float16"])
def test_dump_byte_identical_to_reference_exporter(tmp_path, dtype):
    out = tmp_path / "cap.dpkv"
    man = C.export("synthetic-llama", PROMPT, STEPS, out, dtype=dtype, seed=0, prompt_source="golden", device="cpu")
    gold = os.path.join(GOLDEN, f"pyexport_synth_{dtype}.dpkv")
    with open(out, "rb") as f, open(gold, "rb") as g:
        assert f.read() == g.read()
    with open(str(out) + ".manifest.json") as f, open(gold + ".manifest.json") as g:
        mine, ref = json.load(f), json.load(g)
    mine.pop("dump_path"), ref.pop("dump_path")
    assert mine == ref
    assert man.query_scale == [1.0] * man.num_layers and man.gqa_group == 2


def test_export_errors_leave_no_files(tmp_path):
    out = tmp_path / "x.dpkv"
    with pytest.raises(C.ExportError, match="empty"):
        C.export("synthetic-llama", "", 2, out, device="cpu")
    with pytest.raises(C.ExportError, match="positions"):
        C.export("synthetic-llama", "x" * 500, 20, out, device="cpu")
    with pytest.raises(C.ExportError, match="out of range"):
        C.export("synthetic-llama", PROMPT, 2, out, layers=[0, 5], device="cpu")
    with pytest.raises(C.ExportError, match="steps"):
        C.export("synthetic-llama", PROMPT, 0, out, device="cpu")
    assert not os.listdir(tmp_path)


def test_layer_subset_and_cli(tmp_path, capsys):
    pf = tmp_path / "p.txt"
    pf.write_text(PROMPT)
    out = tmp_path / "sub.dpkv"
    assert C.main(["--prompt-file", str(pf), "--steps", "3", "--layers", "1", "--out", str(out),
                   "--device", "cpu"]) == 0
    txt = capsys.readouterr().out
    assert "1 layers, 4 query heads" in txt and "manifest.json" in txt
    with open(str(out) + ".manifest.json") as f:
        assert json.load(f)["layers_exported"] == [1]
    assert C.main(["--prompt-file", str(tmp_path / "missing.txt"), "--out", str(out)]) == 1
    assert capsys.readouterr().err.startswith("pyexport: error:")


def test_run_greedy_probabilities_cover_growing_prefix():
    model = C.build_synthetic_model(seed=0)
    cap = C.run_greedy(model, C.encode_bytes(PROMPT), 3, keep_probabilities=True)
    for s, rows in enumerate(cap.probabilities):
        assert tuple(rows.shape) == (2, 4, cap.prompt_len + s + 1)
        assert torch.allclose(rows.sum(-1), torch.ones(()), atol=1e-5)
    with pytest.raises(ValueError):
        C.run_greedy(model, [], 1)
    with pytest.raises(ValueError):
        C.run_greedy(model, [1, 2], 0)


LONG = " ".join([PROMPT] * 3)  # ~420 tokens: a few dozen clusters per head


@pytest.mark.gpu
def test_device_capture_decode_parity_and_runtime_round_trip():
    from oracle import doublep_oracle as O

    import paper_2602_05191_b200 as P

    model = C.build_synthetic_model(seed=0, device="cuda")
    cap = C.run_greedy(model, C.encode_bytes(LONG), 8, keep_probabilities=True)
    assert cap.keys.is_cuda and cap.queries.is_cuda
    cache, trace = cap.device_cache()
    cc = P.build_clustered_cache(cache, sink=4, window=64, tokens_per_cluster=8, seed=0)
    cfg = P.DoublePConfig(0.95, 0.7)
    keys = cache.keys.double().cpu().numpy()[..., :cache.head_dim]
    values = cache.values.double().cpu().numpy()[..., :cache.head_dim]
    worst_out = worst_rt = 0.0
    n_exact = 0
    for layer in range(cap.num_layers):
        for hq in range(trace.num_query_heads):
            h = trace.kv_head_for(hq)
            t = cc.estimation_data(layer, h)
            tables = O.HeadTables(members=t["members"], centroids=t["centroids"], value_means=t["value_means"])
            for s in range(trace.num_steps):
                q = trace.query(s, layer, hq)
                out, plan, est = P.decode_step(q, cache, cc, cfg, layer, h)
                ref, oplan, oest = O.decode_step(q.astype(np.float64), keys[layer, h], values[layer, h], tables,
                                                 0.95, 0.7, 4, 64)
                assert np.max(np.abs(est.log_masses - oest.log_masses)) <= 1e-9
                if np.array_equal(plan.exact_tokens, oplan.exact_tokens):
                    n_exact += 1
                else:  # allowed only at a score tie
                    lm = np.sort(oest.log_masses)[::-1]
                    assert np.min(np.abs(np.diff(lm))) <= 1e-6
                worst_out = max(worst_out, O.output_error(out.output, ref.output))
                w, _ = P.full_attention_weights(q, cache, layer, h)
                worst_rt = max(worst_rt, float(np.abs(w - cap.prefix_probabilities(s, layer, hq)).max()))
    total = cap.num_layers * trace.num_query_heads * trace.num_steps
    print(f"\n[CAPTURE] synthetic-llama on cuda: {total} (layer, head, step) decodes, exact sets {n_exact}, "
          f"worst out err {worst_out:.1e}, worst |w - runtime| {worst_rt:.1e}")
    assert worst_out <= 1e-5
    assert worst_rt <= 1e-5
