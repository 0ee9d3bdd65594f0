"""Capture real attention tensors from a transformers model during greedy
decode -- the reference's `pyexport` (pkg/pyexport/src/pyexport/capture.py,
exporter.py, cli.py) on the B200 path.

The model runs where its weights live (a CUDA device here), so the captured
keys and values are already device tensors: ``GenerationCapture.device_cache``
hands them to the clustered-cache build without a host round trip, and
``export`` writes the same DPKV dump + JSON manifest the reference writes
(byte-identical for the same model, prompt, steps and dtype: see
tests/test_capture.py against the reference's own dump).

What is recorded, per layer (reference semantics, capture.py:1-16):
  * the post-rotary keys and values the prefill forward caches -- read
    straight from the model's KV cache object after the prefill;
  * one post-rotary query per query head per greedy step -- taken on the way
    through a registered attention implementation that delegates to the stock
    eager path (outputs unchanged);
  * optionally the runtime's own softmax probabilities (the round-trip
    oracle).
Queries are exported pre-multiplied by ``scaling * sqrt(head_dim)`` so the
fixed ``q.k / sqrt(d)`` logit convention reproduces the runtime's logits
(exporter.py:145-148; the factor is 1 for Llama).

    python -m paper_2602_05191_b200.capture --model synthetic-llama \\
        --prompt-file prompt.txt --steps 16 --out cap.dpkv [--device cuda]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import tempfile
from dataclasses import asdict, dataclass

import numpy as np
import torch

SYNTHETIC_MODEL_ID = "synthetic-llama"
ATTN_IMPLEMENTATION = "b200-capture"
# the reference's download-free model (capture.py:34-56): GQA, two layers,
# byte-level vocabulary so raw prompt bytes are token ids
SYNTHETIC_GEOMETRY = dict(hidden_size=64, num_attention_heads=4, num_key_value_heads=2, num_hidden_layers=2,
                          intermediate_size=128, vocab_size=256, max_position_embeddings=512)
DTYPES = {"float32": torch.float32, "float16": torch.float16, "bfloat16": torch.bfloat16}


class CaptureError(RuntimeError):
    """Recorded tensors do not line up with the model geometry (capture.py:59-60)."""


class ExportError(RuntimeError):
    """An export could not be completed; no partial files remain (exporter.py:24-25)."""


def build_synthetic_model(seed=0, dtype=torch.float32, device="cpu"):
    """Deterministically initialised small Llama (random weights)."""
    from transformers import LlamaConfig, LlamaForCausalLM

    torch.manual_seed(seed)
    model = LlamaForCausalLM(LlamaConfig(**SYNTHETIC_GEOMETRY))  # initialised on the host: same weights anywhere
    return model.to(dtype).to(device).eval()


def encode_bytes(text):
    return list(text.encode("utf-8"))


class _Tap:
    """Receives every attention call of the wrapped model."""

    def __init__(self, keep_probabilities):
        self.keep = keep_probabilities
        self.decoding = False
        self.prefill_seen = set()
        self.steps = []        # per decode forward: {layer: (query [Hq, d], probs [Hq, T] or None)}
        self.scaling = {}

    def __call__(self, layer, query, weights, scaling):
        self.scaling[layer] = float(scaling)
        if not self.decoding:
            if layer in self.prefill_seen:
                raise CaptureError(f"layer {layer} seen twice during prefill")
            self.prefill_seen.add(layer)
            return
        step = self.steps[-1]
        if layer in step:
            raise CaptureError(f"layer {layer} seen twice in one decode step")
        probs = None
        if self.keep:
            if weights is None:
                raise CaptureError("runtime returned no attention weights to record")
            probs = weights[0, :, 0, :].detach().float()
        step[layer] = (query[0, :, 0, :].detach().float(), probs)


_TAP = None


def _tap_forward(module, query, key, value, attention_mask, scaling=None, dropout=0.0, **kwargs):
    from transformers.models.llama.modeling_llama import eager_attention_forward

    out, weights = eager_attention_forward(module, query, key, value, attention_mask, scaling, dropout=dropout,
                                           **kwargs)
    if _TAP is not None:
        _TAP(module.layer_idx, query, weights, scaling if scaling is not None else module.scaling)
    return out, weights


def _register():
    from transformers import AttentionInterface

    AttentionInterface.register(ATTN_IMPLEMENTATION, _tap_forward)


@dataclass(frozen=True)
class GenerationCapture:
    """One greedy run (capture.py:137-184).  keys/values [L, Hkv, P, d] and
    queries [S, L, Hq, d] are float32 tensors on the model's device;
    probabilities (optional) one [L, Hq, P + s + 1] tensor per step."""

    prompt_len: int
    num_layers: int
    num_kv_heads: int
    num_query_heads: int
    head_dim: int
    keys: torch.Tensor
    values: torch.Tensor
    queries: torch.Tensor
    scaling: np.ndarray
    probabilities: list | None
    generated_ids: list

    @property
    def num_steps(self):
        return self.queries.shape[0]

    @property
    def gqa_group(self):
        return self.num_query_heads // self.num_kv_heads

    def prefix_probabilities(self, step, layer, query_head):
        """The runtime's attention over the prompt columns, renormalised
        (the distribution a dense recomputation from the dump reproduces)."""
        if self.probabilities is None:
            raise CaptureError("probabilities were not recorded")
        row = self.probabilities[step][layer, query_head, :self.prompt_len].double().cpu().numpy()
        total = float(row.sum())
        if total <= 0.0:
            raise CaptureError("no attention mass on the prompt columns")
        return row / total

    def export_queries(self, layers=None):
        """Queries with the runtime's scaling baked in (exporter.py:145-148)."""
        sel = list(range(self.num_layers)) if layers is None else list(layers)
        scale = self.scaling[sel] * math.sqrt(self.head_dim)  # float64, as the reference multiplies
        sd = torch.from_numpy(scale).to(self.queries.device)
        return (self.queries[:, sel].double() * sd[None, :, None, None]).float(), scale

    def device_cache(self, layers=None, device="cuda"):
        """(KvCache, QueryTrace) of this package for the selected layers, built
        from the captured device tensors (no host round trip of the KV)."""
        from .cache import KvCache, QueryTrace

        sel = list(range(self.num_layers)) if layers is None else list(layers)
        q, _ = self.export_queries(sel)
        return (KvCache(self.keys[sel].to(device), self.values[sel].to(device)),
                QueryTrace(queries=q, gqa_group=self.gqa_group))


def run_greedy(model, input_ids, steps, keep_probabilities=False):
    """``steps`` greedy decode forwards after one prefill forward
    (capture.py:187-228).  Keys/values come from the prefill's KV cache;
    queries (and optionally probabilities) from the attention tap."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    ids = torch.as_tensor(list(input_ids), dtype=torch.long)
    if ids.ndim != 1 or ids.numel() == 0:
        raise ValueError("input_ids must be a nonempty 1-D sequence")
    dev = next(model.parameters()).device
    _register()
    tap = _Tap(keep_probabilities)
    previous = model.config._attn_implementation
    model.set_attn_implementation(ATTN_IMPLEMENTATION)
    global _TAP
    _TAP = tap
    fed = []
    try:
        with torch.no_grad():
            out = model(ids.unsqueeze(0).to(dev), use_cache=True)
            past = out.past_key_values
            kv = _cache_tensors(past)  # post-rotary prefill K/V, snapshotted before decode appends
            nxt = int(out.logits[0, -1].argmax())
            tap.decoding = True
            for _ in range(steps):
                tap.steps.append({})
                fed.append(nxt)
                out = model(torch.tensor([[nxt]], dtype=torch.long, device=dev), past_key_values=past,
                            use_cache=True)
                past = out.past_key_values
                nxt = int(out.logits[0, -1].argmax())
    finally:
        _TAP = None
        model.set_attn_implementation(previous)
    return _assemble(tap, kv, int(ids.numel()), fed)


def _cache_tensors(past):
    layers = getattr(past, "layers", None)
    if layers is not None:  # transformers >= 4.56 DynamicCache
        pairs = [(lay.keys, lay.values) for lay in layers]
    else:
        pairs = list(zip(past.key_cache, past.value_cache))
    return [(k[0].detach().float().clone(), v[0].detach().float().clone()) for k, v in pairs]


def _assemble(tap, kv, prompt_len, fed):
    if not tap.prefill_seen:
        raise CaptureError("no attention calls recorded during prefill")
    layer_ids = sorted(tap.prefill_seen)
    if layer_ids != list(range(len(layer_ids))) or len(kv) != len(layer_ids):
        raise CaptureError(f"non-contiguous layer indices {layer_ids}")
    keys = torch.stack([k for k, _ in kv])
    values = torch.stack([v for _, v in kv])
    if keys.shape != values.shape:
        raise CaptureError(f"key/value shape mismatch: {tuple(keys.shape)} vs {tuple(values.shape)}")
    L, H, n, d = keys.shape
    if n != prompt_len:
        raise CaptureError(f"prefill cached {n} positions for a {prompt_len}-token prompt")
    queries, probs = [], ([] if tap.keep else None)
    for i, step in enumerate(tap.steps):
        if sorted(step) != layer_ids:
            raise CaptureError(f"decode step {i} covered layers {sorted(step)}, expected {layer_ids}")
        queries.append(torch.stack([step[li][0] for li in layer_ids]))
        if probs is not None:
            rows = torch.stack([step[li][1] for li in layer_ids])
            if rows.shape[-1] != prompt_len + i + 1:
                raise CaptureError(f"step {i} attention spans {rows.shape[-1]} columns, expected "
                                   f"{prompt_len + i + 1}")
            probs.append(rows)
    queries = torch.stack(queries)
    Hq = queries.shape[2]
    if queries.shape[3] != d:
        raise CaptureError(f"query head_dim {queries.shape[3]} != key head_dim {d}")
    if Hq % H:
        raise CaptureError(f"{Hq} query heads not divisible by {H} kv heads")
    return GenerationCapture(prompt_len=prompt_len, num_layers=L, num_kv_heads=H, num_query_heads=Hq, head_dim=d,
                             keys=keys, values=values, queries=queries,
                             scaling=np.array([tap.scaling[li] for li in layer_ids]), probabilities=probs,
                             generated_ids=fed)


@dataclass(frozen=True)
class ExportManifest:
    """Provenance of one dump (exporter.py:35-59); the num_*/context fields
    match the DPKV header."""

    model: str
    prompt_source: str
    layers_exported: list
    query_heads_exported: list
    num_layers: int
    num_kv_heads: int
    num_query_heads: int
    head_dim: int
    context_len: int
    num_steps: int
    gqa_group: int
    source_dtype: str
    query_scale: list
    dump_path: str

    def to_dict(self):
        return asdict(self)


def _load(model_id, dtype, seed, prompt, device):
    if model_id == SYNTHETIC_MODEL_ID:
        return build_synthetic_model(seed=seed, dtype=dtype, device=device), encode_bytes(prompt)
    from transformers import AutoModelForCausalLM, AutoTokenizer

    try:
        tok = AutoTokenizer.from_pretrained(model_id)
        model = AutoModelForCausalLM.from_pretrained(model_id, dtype=dtype).to(device).eval()
    except Exception as exc:
        raise ExportError(f"cannot load model {model_id!r}: {exc}") from exc
    return model, tok.encode(prompt)


def _atomic_json(payload, path):
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path) or ".", suffix=".json.tmp")
    try:
        with os.fdopen(fd, "w", encoding="utf-8") as fh:
            json.dump(payload, fh, indent=2)
            fh.write("\n")
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def export(model_id, prompt, steps, out_path, *, layers=None, dtype="float32", seed=0, prompt_source="<inline>",
           device="cpu"):
    """Greedy decode on ``model_id`` and write the DPKV dump plus
    ``<out>.manifest.json`` (exporter.py:107-175).  Returns the manifest;
    on failure no output file is left behind."""
    from .dpkv import write_dpkv

    if steps < 1:
        raise ExportError("steps must be >= 1")
    if dtype not in DTYPES:
        raise ExportError(f"unknown dtype {dtype!r}; choose from {sorted(DTYPES)}")
    model, ids = _load(model_id, DTYPES[dtype], seed, prompt, device)
    if len(ids) == 0:
        raise ExportError("prompt is empty")
    maxpos = int(model.config.max_position_embeddings)
    if len(ids) + steps > maxpos:
        raise ExportError(f"prompt ({len(ids)} tokens) plus {steps} steps exceeds the model's {maxpos} positions")
    cap = run_greedy(model, ids, steps)
    if layers is None:
        sel = list(range(cap.num_layers))
    else:
        sel = sorted(set(int(x) for x in layers))
        if not sel:
            raise ExportError("layer selection is empty")
        bad = [x for x in sel if x < 0 or x >= cap.num_layers]
        if bad:
            raise ExportError(f"layer selection {bad} out of range for a {cap.num_layers}-layer model")
    q, scale = cap.export_queries(sel)
    keys, values, qn = (t.cpu().numpy() for t in (cap.keys[sel], cap.values[sel], q))
    if not (np.isfinite(keys).all() and np.isfinite(values).all() and np.isfinite(qn).all()):
        raise ExportError("captured tensors are inconsistent: non-finite entries")
    out_path = os.fspath(out_path)
    man = ExportManifest(model=model_id, prompt_source=prompt_source, layers_exported=sel,
                         query_heads_exported=list(range(cap.num_query_heads)), num_layers=len(sel),
                         num_kv_heads=cap.num_kv_heads, num_query_heads=cap.num_query_heads, head_dim=cap.head_dim,
                         context_len=cap.prompt_len, num_steps=cap.num_steps, gqa_group=cap.gqa_group,
                         source_dtype=dtype, query_scale=[float(x) for x in scale],
                         dump_path=out_path)
    write_dpkv(out_path, keys, values, qn)
    _atomic_json(man.to_dict(), f"{out_path}.manifest.json")
    return man


def main(argv=None):
    """`pyexport` CLI (cli.py:1-86): same flags, messages and exit codes, plus --device."""
    p = argparse.ArgumentParser(prog="pyexport", description="Export attention tensors from a greedy decode run "
                                "into a DPKV dump plus JSON manifest.")
    p.add_argument("--model", default=SYNTHETIC_MODEL_ID)
    p.add_argument("--prompt-file", required=True)
    p.add_argument("--steps", type=int, default=16)
    p.add_argument("--layers", default=None, help="comma-separated layer indices (default: all)")
    p.add_argument("--dtype", choices=tuple(DTYPES), default="float32")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True)
    p.add_argument("--device", default="cuda" if torch.cuda.is_available() else "cpu")
    a = p.parse_args(argv)
    try:
        layers = None
        if a.layers is not None:
            try:
                layers = [int(t) for t in a.layers.split(",") if t.strip() != ""]
            except ValueError:
                raise ExportError(f"bad layer list {a.layers!r}") from None
        with open(a.prompt_file, encoding="utf-8") as fh:
            prompt = fh.read()
        man = export(a.model, prompt, a.steps, a.out, layers=layers, dtype=a.dtype, seed=a.seed,
                     prompt_source=a.prompt_file, device=a.device)
    except Exception as exc:
        print(f"pyexport: error: {exc}", file=sys.stderr)
        return 1
    print(f"wrote {man.dump_path}: {man.num_layers} layers, {man.num_query_heads} query heads, context "
          f"{man.context_len}, {man.num_steps} steps")
    print(f"wrote {man.dump_path}.manifest.json")
    return 0


if __name__ == "__main__":
    sys.exit(main())
