"""DPKV ingest: the device loader against a file written by
the REAL reference (tests/golden/ref_small.dpkv, oracle/gen_golden_dpkv.py),
the reference's validation errors, and the decode path on ingested caches."""

import os
import shutil
import struct

import numpy as np
import pytest
import torch

from paper_2602_05191_b200 import dpkv

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ref():
    return np.load(os.path.join(GOLD, "ref_small_dpkv.npz"))


def test_reads_reference_written_file_exactly():
    ref = _ref()
    hdr, ks, vs, q = dpkv.load_dpkv(os.path.join(GOLD, "ref_small.dpkv"), device="cpu", dtype=torch.float32)
    assert (hdr.num_layers, hdr.num_kv_heads, hdr.context_len, hdr.head_dim) == ref["keys"].shape
    assert hdr.gqa_group == int(ref["gqa_group"])
    for li in range(hdr.num_layers):
        assert np.array_equal(ks[li][0].numpy(), ref["keys"][li])
        assert np.array_equal(vs[li][0].numpy(), ref["values"][li])
    assert np.array_equal(np.asarray(q), ref["queries"])


def test_writer_round_trip_is_byte_identical(tmp_path):
    ref = _ref()
    out = tmp_path / "rt.dpkv"
    dpkv.write_dpkv(out, ref["keys"], ref["values"], ref["queries"])
    with open(out, "rb") as a, open(os.path.join(GOLD, "ref_small.dpkv"), "rb") as b:
        assert a.read() == b.read()


def _corrupt(tmp_path, fn):
    p = tmp_path / "bad.dpkv"
    shutil.copy(os.path.join(GOLD, "ref_small.dpkv"), p)
    blob = bytearray(open(p, "rb").read())
    blob = fn(blob)
    open(p, "wb").write(bytes(blob))
    return p


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXX" + b[4:], "not a DPKV file"),
    (lambda b: b[:10], "truncated file"),
    (lambda b: b[:-5], "truncated file"),
    (lambda b: b + b"\0", "trailing bytes after trailer"),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "unsupported version 2"),
    (lambda b: b[:40] + bytes([b[40] ^ 0xFF]) + b[41:], "corrupt payload"),
    (lambda b: b[:8] + struct.pack("<I", 0) + b[12:], "invalid header: num_layers = 0"),
])
def test_reference_error_messages(tmp_path, mutate, msg):
    p = _corrupt(tmp_path, mutate)
    with pytest.raises(dpkv.DumpFormatError, match=msg):
        dpkv.load_dpkv(p, device="cpu")


@pytest.mark.gpu
def test_ingested_cache_through_the_decode_path():
    """A reference-written capture, uploaded to the GPU, clustered and decoded:
    the sparse step at p1 = p2 = 1 equals the dense kernel (exactness collapse)."""
    from paper_2602_05191_b200 import cluster_layer, dense_attention, sparse_attention

    hdr, ks, vs, q = dpkv.load_dpkv(os.path.join(GOLD, "ref_small.dpkv"), dtype=torch.float32)
    for li in range(hdr.num_layers):
        layer = cluster_layer(ks[li], vs[li], layer=li)
        qs = torch.from_numpy(np.array(q[0, li])).cuda().unsqueeze(0)
        sp = sparse_attention(qs, layer, 1.0, 1.0).clone()
        de = dense_attention(qs, layer).clone()
        err = ((sp - de).norm(dim=-1) / de.norm(dim=-1)).max().item()
        assert err <= 1e-5, err
