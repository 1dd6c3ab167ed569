"""HPDR multi-chunk container.

The reference package defines the format only in its SPEC.  With pipeline id 2 every chunk
payload is a reference-identical MGARD blob of one dim-0 slab, compressed with the GLOBAL value
range so the error bound of the whole field holds; with pipeline id 1 every
chunk is a reference-identical fixed-rate stream (hpdr/zfp.py) of its slab.

Layout (little-endian):
  magic "HPDR" | version u16 | pipeline u8 (0 Huffman, 1 ZFP, 2 MGARD) | dtype u8 | rank u8 |
  dims u64 x rank | params (MGARD: eb_rel f64, dict_size u32, global min f64, global max f64;
  ZFP: rate u8) |
  chunk count u32 | per chunk: raw offset u64, raw size u64, payload offset u64, payload size u64 |
  header CRC-32 u32 (of every preceding header byte) | payloads
Offsets are relative to the first payload byte; raw offsets/sizes count elements.
"""
from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field

from .errors import FormatError

MAGIC = b"HPDR"
VERSION = 1
PIPELINE_ZFP = 1
PIPELINE_MGARD = 2


@dataclass
class ChunkEntry:
    raw_offset: int
    raw_size: int
    payload_offset: int
    payload_size: int


@dataclass
class ContainerHeader:
    dtype: int
    dims: tuple
    eb_rel: float
    dict_size: int
    vmin: float
    vmax: float
    chunks: list = field(default_factory=list)
    pipeline: int = PIPELINE_MGARD
    version: int = VERSION
    rate: int = 0   # ZFP containers


def header_bytes(h: ContainerHeader) -> bytes:
    out = bytearray(MAGIC)
    out += struct.pack("<HBBB", h.version, h.pipeline, h.dtype, len(h.dims))
    out += struct.pack(f"<{len(h.dims)}Q", *h.dims)
    if h.pipeline == PIPELINE_ZFP:
        out += struct.pack("<B", h.rate)
    else:
        out += struct.pack("<dIdd", h.eb_rel, h.dict_size, h.vmin, h.vmax)
    out += struct.pack("<I", len(h.chunks))
    for c in h.chunks:
        out += struct.pack("<QQQQ", c.raw_offset, c.raw_size, c.payload_offset, c.payload_size)
    out += struct.pack("<I", zlib.crc32(bytes(out)) & 0xFFFFFFFF)
    return bytes(out)


def write_container(h: ContainerHeader, payloads) -> bytes:
    payloads = [bytes(p) for p in payloads]
    if len(payloads) != len(h.chunks):
        raise FormatError("chunk table and payload count differ")
    off = 0
    for c, p in zip(h.chunks, payloads):
        if c.payload_size != len(p):
            raise FormatError("payload size does not match the chunk table")
        c.payload_offset = off
        off += len(p)
    return header_bytes(h) + b"".join(payloads)


def read_container(data) -> tuple:
    """(header, [payload memoryviews]); raises FormatError on bad magic/version/CRC/truncation."""
    mv = memoryview(data)
    try:
        if bytes(mv[:4]) != MAGIC:
            raise FormatError("bad magic")
        version, pipeline, dtype, rank = struct.unpack_from("<HBBB", mv, 4)
        if version != VERSION:
            raise FormatError(f"unsupported container version {version}")
        if pipeline not in (PIPELINE_MGARD, PIPELINE_ZFP):
            raise FormatError(f"unknown pipeline id {pipeline}")
        pos = 9
        dims = struct.unpack_from(f"<{rank}Q", mv, pos)
        pos += 8 * rank
        eb_rel, dict_size, vmin, vmax, rate = 0.0, 0, 0.0, 0.0, 0
        if pipeline == PIPELINE_ZFP:
            (rate,) = struct.unpack_from("<B", mv, pos)
            pos += 1
        else:
            eb_rel, dict_size, vmin, vmax = struct.unpack_from("<dIdd", mv, pos)
            pos += 28
        (n,) = struct.unpack_from("<I", mv, pos)
        pos += 4
        chunks = []
        for _ in range(n):
            chunks.append(ChunkEntry(*struct.unpack_from("<QQQQ", mv, pos)))
            pos += 32
        (crc,) = struct.unpack_from("<I", mv, pos)
    except struct.error as e:
        raise FormatError(f"truncated container header: {e}") from e
    if zlib.crc32(bytes(mv[:pos])) & 0xFFFFFFFF != crc:
        raise FormatError("header checksum mismatch")
    pos += 4
    h = ContainerHeader(dtype, tuple(dims), eb_rel, dict_size, vmin, vmax, chunks, pipeline, version, rate)
    payloads = []
    prev = -1
    for c in chunks:
        if c.payload_size:   # empty payloads occupy no bytes (their offset repeats the next one)
            if c.payload_offset <= prev:
                raise FormatError("payload offsets not strictly increasing")
            prev = c.payload_offset
        a, b = pos + c.payload_offset, pos + c.payload_offset + c.payload_size
        if b > len(mv):
            raise FormatError("container truncated in payloads")
        payloads.append(mv[a:b])
    return h, payloads


def slab_bounds(n0: int, parts: int, index: int) -> tuple:
    """[start, stop) planes of slab ``index`` when n0 planes split into ``parts`` (stages.py:99-103)."""
    base, rem = divmod(n0, parts)
    start = index * base + min(index, rem)
    return start, start + base + (1 if index < rem else 0)
