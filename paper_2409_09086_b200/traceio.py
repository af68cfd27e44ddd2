"""Reader for the reference's binary attention-trace format (``.imtrace``,
reference traceio.py:1-14, 98-184): the input of the device trace replay.

Host-side parsing only (the format is I/O, not compute).  Same event types,
validation (ATTN_ROW sums within 1e-3, n non-decreasing within a round) and
``TraceFormatError`` with the failing byte offset as the reference.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import BinaryIO, Iterator, List, Optional, Tuple

import numpy as np

F32 = np.float32
MAGIC = b"IMT1"
VERSION = 1
FLAG_HEAD_AGGREGATED = 1
TAG_ROUND_START, TAG_TOKENS, TAG_ATTN_ROW, TAG_SADDLE_TRUTH = 1, 2, 3, 4
HEADER_STRUCT = struct.Struct("<4sIIII")
ROW_SUM_TOLERANCE = 1e-3


class TraceFormatError(Exception):
    """Malformed trace data (traceio.py:47-54)."""

    def __init__(self, message: str, offset: Optional[int] = None):
        if offset is not None:
            message = f"{message} (byte offset {offset})"
        super().__init__(message)
        self.offset = offset


@dataclass(frozen=True)
class TraceHeader:
    layers: int
    heads: int
    flags: int = FLAG_HEAD_AGGREGATED
    version: int = VERSION


@dataclass(frozen=True)
class RoundStart:
    round_id: int
    prompt_len: int


@dataclass(frozen=True, eq=False)
class Tokens:
    modality: np.ndarray


@dataclass(frozen=True, eq=False)
class AttnRow:
    layer: int
    probs: np.ndarray


@dataclass(frozen=True, eq=False)
class SaddleTruth:
    round_id: int
    ids: np.ndarray


def _read_exact(source: BinaryIO, size: int, offset: int, what: str) -> bytes:
    data = source.read(size)
    if len(data) != size:
        raise TraceFormatError(f"truncated {what}: wanted {size} bytes, got {len(data)}", offset)
    return data


def read_header(source: BinaryIO) -> TraceHeader:
    magic, version, layers, heads, flags = HEADER_STRUCT.unpack(_read_exact(source, HEADER_STRUCT.size, 0, "header"))
    if magic != MAGIC:
        raise TraceFormatError(f"bad magic {magic!r}, expected {MAGIC!r}", 0)
    if version != VERSION:
        raise TraceFormatError(f"unsupported version {version}, expected {VERSION}", 4)
    return TraceHeader(layers=layers, heads=heads, flags=flags, version=version)


def read_trace(source: BinaryIO, strict: bool = True) -> Tuple[TraceHeader, Iterator]:
    header = read_header(source)

    def events():
        offset = HEADER_STRUCT.size
        last_n = 0
        while True:
            tag_byte = source.read(1)
            if not tag_byte:
                return
            tag, start = tag_byte[0], offset
            offset += 1
            if tag == TAG_ROUND_START:
                round_id, prompt_len = struct.unpack("<II", _read_exact(source, 8, offset, "ROUND_START"))
                offset += 8
                last_n = 0
                yield RoundStart(round_id, prompt_len)
            elif tag == TAG_TOKENS:
                (count,) = struct.unpack("<I", _read_exact(source, 4, offset, "TOKENS count"))
                offset += 4
                body = _read_exact(source, count, offset, "TOKENS modality bytes")
                offset += count
                yield Tokens(np.frombuffer(body, dtype=np.uint8).copy())
            elif tag == TAG_ATTN_ROW:
                layer, n = struct.unpack("<II", _read_exact(source, 8, offset, "ATTN_ROW header"))
                offset += 8
                probs = np.frombuffer(_read_exact(source, 4 * n, offset, "ATTN_ROW probabilities"), "<f4").astype(F32)
                if strict:
                    total = float(probs.sum(dtype=np.float64))
                    if abs(total - 1.0) > ROW_SUM_TOLERANCE:
                        raise TraceFormatError(f"ATTN_ROW sums to {total:.6f}, expected 1 +/- {ROW_SUM_TOLERANCE}", start)
                    if n < last_n:
                        raise TraceFormatError(f"ATTN_ROW n decreased within a round ({n} < {last_n})", start)
                last_n = max(last_n, n)
                offset += 4 * n
                yield AttnRow(layer, probs)
            elif tag == TAG_SADDLE_TRUTH:
                round_id, count = struct.unpack("<II", _read_exact(source, 8, offset, "SADDLE_TRUTH header"))
                offset += 8
                body = _read_exact(source, 4 * count, offset, "SADDLE_TRUTH ids")
                offset += 4 * count
                yield SaddleTruth(round_id, np.frombuffer(body, dtype="<u4").copy())
            else:
                raise TraceFormatError(f"unknown event tag {tag}", start)

    return header, events()


def read_trace_file(path, strict: bool = True) -> Tuple[TraceHeader, List]:
    with open(path, "rb") as fh:
        header, it = read_trace(fh, strict=strict)
        return header, list(it)
