"""DPKV dump ingest: a reference (cache, trace) file straight into device layers.

The reference's capture/export path (pyexport, ``kvcache.write_dump``,
kvcache.py:156-192) stores real attention K/V and query traces in the DPKV
format:

    b"DPKV" | u32 version (1) | <6I header: layers, kv_heads, q_heads,
    head_dim, context_len, steps | f32 K/V blocks [layer][kv head][K, V]
    [context_len, head_dim] | f32 queries [steps, layers, q_heads, head_dim] |
    u32 CRC-32 of everything after the header

``read_dump`` (kvcache.py:195-255) loads the whole file into host memory and
validates it.  Here the file is memory-mapped, the CRC is checked in
streaming chunks, and each layer's K/V go to the GPU one layer at a time in
the decode layout ([B=1, H, N, d], bf16 or fp32), so a multi-GB capture never
needs a second host copy.  The same validation order and error messages as
``read_dump`` apply (``DumpFormatError`` is a ``ValueError``).
"""

from __future__ import annotations

import os
import struct
import zlib
from dataclasses import dataclass

import numpy as np

MAGIC = b"DPKV"
VERSION = 1
_HEADER = struct.Struct("<6I")
_CRC_CHUNK = 64 << 20


class DumpFormatError(ValueError):
    """Malformed DPKV file (mirror of doublep.kvcache.DumpFormatError)."""


@dataclass(frozen=True)
class DpkvHeader:
    num_layers: int
    num_kv_heads: int
    num_query_heads: int
    head_dim: int
    context_len: int
    num_steps: int

    @property
    def gqa_group(self) -> int:
        return self.num_query_heads // self.num_kv_heads

    @property
    def kv_bytes(self) -> int:
        return self.num_layers * self.num_kv_heads * 2 * self.context_len * self.head_dim * 4

    @property
    def q_bytes(self) -> int:
        return self.num_steps * self.num_layers * self.num_query_heads * self.head_dim * 4


def _open_checked(path, verify_crc=True):
    """Validate like read_dump (kvcache.py:201-240); returns (header, memmap)."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(8 + _HEADER.size)
    if len(head) < 4 or head[:4] != MAGIC:
        raise DumpFormatError("not a DPKV file")
    if len(head) < 8 + _HEADER.size:
        raise DumpFormatError("truncated file")
    (version,) = struct.unpack_from("<I", head, 4)
    if version != VERSION:
        raise DumpFormatError(f"unsupported version {version}")
    vals = _HEADER.unpack_from(head, 8)
    layers, kv_heads, q_heads, dim, context, steps = vals
    for name, val in (("num_layers", layers), ("num_kv_heads", kv_heads), ("num_query_heads", q_heads),
                      ("head_dim", dim), ("context_len", context)):
        if val < 1:
            raise DumpFormatError(f"invalid header: {name} = {val}")
    if kv_heads > q_heads or q_heads % kv_heads != 0:
        raise DumpFormatError(
            f"invalid header: num_query_heads {q_heads} not a multiple of num_kv_heads {kv_heads}")
    hdr = DpkvHeader(*vals)
    body = 8 + _HEADER.size
    expected = body + hdr.kv_bytes + hdr.q_bytes + 4
    if size < expected:
        raise DumpFormatError("truncated file")
    if size > expected:
        raise DumpFormatError("trailing bytes after trailer")
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    if verify_crc:
        crc = 0
        end = expected - 4
        for off in range(body, end, _CRC_CHUNK):
            crc = zlib.crc32(mm[off:min(end, off + _CRC_CHUNK)], crc)
        (stored,) = struct.unpack("<I", bytes(mm[end:expected]))
        if crc != stored:
            raise DumpFormatError("corrupt payload")
    return hdr, mm


def read_header(path) -> DpkvHeader:
    """Header of a DPKV file (validated, payload not read)."""
    return _open_checked(path, verify_crc=False)[0]


def load_dpkv(path, device="cuda", dtype=None, layers=None, verify_crc=True):
    """Load a DPKV dump for the device decode path.

    Returns (header, keys, values, queries): keys/values are lists (one per
    selected layer) of [1, H, N, d] tensors on `device` (dtype defaults to
    torch.bfloat16; torch.float32 keeps the file's exact values), queries a
    read-only float32 view [steps, layers, Hq, d] of the file.  Layers are
    uploaded one at a time from the memory map."""
    import torch

    dtype = torch.bfloat16 if dtype is None else dtype
    hdr, mm = _open_checked(path, verify_crc)
    body = 8 + _HEADER.size
    kv = np.ndarray((hdr.num_layers, hdr.num_kv_heads, 2, hdr.context_len, hdr.head_dim), dtype="<f4",
                    buffer=mm, offset=body)
    q = np.ndarray((hdr.num_steps, hdr.num_layers, hdr.num_query_heads, hdr.head_dim), dtype="<f4", buffer=mm,
                   offset=body + hdr.kv_bytes)
    sel = range(hdr.num_layers) if layers is None else list(layers)
    if not np.isfinite(q).all():
        raise DumpFormatError("invalid payload: queries must be finite")
    keys, values = [], []
    for li in sel:
        blk = torch.from_numpy(np.array(kv[li]))  # [H, 2, N, d] f32 (one layer, copied out of the map)
        if not torch.isfinite(blk).all():
            raise DumpFormatError("invalid payload: keys/values must be finite")
        blk = blk.to(device)
        keys.append(blk[:, 0].to(dtype).unsqueeze(0).contiguous())
        values.append(blk[:, 1].to(dtype).unsqueeze(0).contiguous())
    return hdr, keys, values, q


def write_dpkv(path, keys, values, queries):
    """Write a DPKV file (write_dump's format, kvcache.py:156-192) from host
    arrays: keys/values [L, Hkv, N, d], queries [S, L, Hq, d]; atomic rename."""
    keys = np.asarray(keys, dtype="<f4")
    values = np.asarray(values, dtype="<f4")
    queries = np.asarray(queries, dtype="<f4")
    L, H, N, d = keys.shape
    S, _, Hq, _ = queries.shape
    tmp = os.fspath(path) + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<I", VERSION))
        fh.write(_HEADER.pack(L, H, Hq, d, N, S))
        crc = 0
        for li in range(L):
            for h in range(H):
                for blk in (keys[li, h], values[li, h]):
                    b = np.ascontiguousarray(blk).tobytes()
                    crc = zlib.crc32(b, crc)
                    fh.write(b)
        b = np.ascontiguousarray(queries).tobytes()
        crc = zlib.crc32(b, crc)
        fh.write(b)
        fh.write(struct.pack("<I", crc))
    os.replace(tmp, path)
