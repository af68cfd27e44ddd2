"""The reference's binary attention-trace format (``.imtrace``; layout at
/root/reference/pkg/src/streamkv/traceio.py:1-14): the input of the batched
device replay (``replay.py``).

Layout, little-endian: a 20-byte header (magic "IMT1", version 1, layers,
heads, flags), then tagged records -- ROUND_START(round, prompt_len),
TOKENS(count, count bytes), ATTN_ROW(layer, n, n float32),
SADDLE_TRUTH(round, count, count u32).

The file is read into memory once and indexed by a single record scan
(``TraceIndex``): every ATTN_ROW payload becomes a slice of one flat float32
array that the replay uploads to the GPU in one copy, with per-row layer /
offset / length columns.  The event objects of the reference API
(``read_trace``) are views built from that index.  Validation matches the
reference reader: strict mode checks that each row sums to 1 within 1e-3 and
that n does not decrease within a round; errors are ``TraceFormatError``
carrying the byte offset of the failing record (or of the truncated field).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import BinaryIO, Iterator, List, Optional, Tuple

import numpy as np

F32 = np.float32
MAGIC = b"IMT1"
VERSION = 1
FLAG_HEAD_AGGREGATED = 1
TAG_ROUND_START, TAG_TOKENS, TAG_ATTN_ROW, TAG_SADDLE_TRUTH = 1, 2, 3, 4
HEADER_STRUCT = struct.Struct("<4sIIII")
ROW_SUM_TOLERANCE = 1e-3

# per tag: (fixed field struct, field label, index of the field that counts the
# body items, body item size, body label)
_RECORDS = {
    TAG_ROUND_START: (struct.Struct("<II"), "ROUND_START", None, 0, ""),
    TAG_TOKENS: (struct.Struct("<I"), "TOKENS count", 0, 1, "TOKENS modality bytes"),
    TAG_ATTN_ROW: (struct.Struct("<II"), "ATTN_ROW header", 1, 4, "ATTN_ROW probabilities"),
    TAG_SADDLE_TRUTH: (struct.Struct("<II"), "SADDLE_TRUTH header", 1, 4, "SADDLE_TRUTH ids"),
}


class TraceFormatError(Exception):
    """Malformed trace data; ``offset`` is the byte position of the failure."""

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


def _need(buf: memoryview, pos: int, size: int, what: str) -> None:
    have = max(0, min(size, len(buf) - pos))
    if have != size:
        raise TraceFormatError(f"truncated {what}: wanted {size} bytes, got {have}", pos)


def parse_header(buf: memoryview) -> TraceHeader:
    _need(buf, 0, HEADER_STRUCT.size, "header")
    magic, version, layers, heads, flags = HEADER_STRUCT.unpack_from(buf, 0)
    if magic != MAGIC:
        raise TraceFormatError(f"bad magic {bytes(magic)!r}, expected {MAGIC!r}", 0)
    if version != VERSION:
        raise TraceFormatError(f"unsupported version {version}, expected {VERSION}", 4)
    return TraceHeader(layers=layers, heads=heads, flags=flags, version=version)


def scan_records(buf: memoryview, strict: bool = True) -> Iterator[tuple]:
    """Yield (tag, record start, fixed fields, body offset, body items) per
    record, validating sizes, tags and (strict) ATTN_ROW invariants."""
    pos = HEADER_STRUCT.size
    end = len(buf)
    last_n = 0
    while pos < end:
        start, tag = pos, buf[pos]
        spec = _RECORDS.get(tag)
        if spec is None:
            raise TraceFormatError(f"unknown event tag {tag}", start)
        fixed, label, count_at, item, body_label = spec
        pos += 1
        _need(buf, pos, fixed.size, label)
        fields = fixed.unpack_from(buf, pos)
        pos += fixed.size
        items = fields[count_at] if count_at is not None else 0
        body = pos
        if items:
            _need(buf, pos, items * item, body_label)
            pos += items * item
        if tag == TAG_ROUND_START:
            last_n = 0
        elif tag == TAG_ATTN_ROW:
            if strict:
                total = float(np.frombuffer(buf, "<f4", items, body).sum(dtype=np.float64))
                if abs(total - 1.0) > ROW_SUM_TOLERANCE:
                    raise TraceFormatError(f"ATTN_ROW sums to {total:.6f}, expected 1 +/- {ROW_SUM_TOLERANCE}",
                                           start)
                if items < last_n:
                    raise TraceFormatError(f"ATTN_ROW n decreased within a round ({items} < {last_n})", start)
            last_n = max(last_n, items)
        yield tag, start, fields, body, items


def _event(buf: memoryview, tag: int, fields: tuple, body: int, items: int):
    if tag == TAG_ROUND_START:
        return RoundStart(fields[0], fields[1])
    if tag == TAG_TOKENS:
        return Tokens(np.frombuffer(buf, np.uint8, items, body).copy())
    if tag == TAG_ATTN_ROW:
        return AttnRow(fields[0], np.frombuffer(buf, "<f4", items, body).astype(F32))
    return SaddleTruth(fields[0], np.frombuffer(buf, "<u4", items, body).copy())


def read_header(source: BinaryIO) -> TraceHeader:
    return parse_header(memoryview(source.read(HEADER_STRUCT.size)))


def read_trace(source: BinaryIO, strict: bool = True) -> Tuple[TraceHeader, Iterator]:
    """Header plus a lazy event iterator (the reference's read_trace contract:
    record errors surface while iterating)."""
    buf = memoryview(source.read())
    header = parse_header(buf)

    def events():
        for tag, _, fields, body, items in scan_records(buf, strict):
            yield _event(buf, tag, fields, body, items)

    return header, events()


def read_trace_file(path, strict: bool = True) -> Tuple[TraceHeader, List]:
    with open(path, "rb") as fh:
        header, it = read_trace(fh, strict=strict)
        return header, list(it)


@dataclass
class TraceIndex:
    """Columnar view of a trace for the device replay.

    ``kind[e]`` is the tag of event e; for ATTN_ROW events ``row[e]`` indexes
    the row columns (``row_layer``, ``row_off`` into ``payload``, ``row_n``);
    ROUND_START events carry (round, prompt_len) in ``round_info[e]``;
    SADDLE_TRUTH events their ids in ``truth[e]``."""

    header: TraceHeader
    kind: np.ndarray
    row: np.ndarray
    round_info: np.ndarray
    row_layer: np.ndarray
    row_off: np.ndarray
    row_n: np.ndarray
    payload: np.ndarray
    truth: dict = field(default_factory=dict)


def index_trace(data, strict: bool = True) -> TraceIndex:
    """One scan of an in-memory trace into a ``TraceIndex``."""
    buf = memoryview(data)
    header = parse_header(buf)
    recs = list(scan_records(buf, strict))
    kinds = np.array([r[0] for r in recs], np.int8)
    row_ev = [i for i, r in enumerate(recs) if r[0] == TAG_ATTN_ROW]
    row = np.full(len(recs), -1, np.int64)
    row[row_ev] = np.arange(len(row_ev))
    n = np.array([recs[i][4] for i in row_ev], np.int64)
    off = np.zeros(len(row_ev), np.int64)
    if len(row_ev):
        off[1:] = np.cumsum(n)[:-1]
    payload = np.empty(int(n.sum()), F32)
    for k, i in enumerate(row_ev):
        payload[off[k]: off[k] + n[k]] = np.frombuffer(buf, "<f4", int(n[k]), recs[i][3])
    info = np.zeros((len(recs), 2), np.int64)
    truth = {}
    for i, (tag, _, fields, body, items) in enumerate(recs):
        if tag == TAG_ROUND_START:
            info[i] = fields
        elif tag == TAG_SADDLE_TRUTH:
            truth[i] = np.frombuffer(buf, "<u4", items, body).astype(np.int64)
    return TraceIndex(header=header, kind=kinds, row=row, round_info=info,
                      row_layer=np.array([recs[i][2][0] for i in row_ev], np.int64), row_off=off,
                      row_n=n.astype(np.int32), payload=payload, truth=truth)


def index_events(header: TraceHeader, events) -> TraceIndex:
    """A ``TraceIndex`` from already-parsed event objects (replay_trace's API)."""
    evs = list(events)
    kinds = np.zeros(len(evs), np.int8)
    row = np.full(len(evs), -1, np.int64)
    info = np.zeros((len(evs), 2), np.int64)
    layers, sizes, chunks, truth = [], [], [], {}
    for i, e in enumerate(evs):
        if isinstance(e, RoundStart):
            kinds[i] = TAG_ROUND_START
            info[i] = (e.round_id, e.prompt_len)
        elif isinstance(e, Tokens):
            kinds[i] = TAG_TOKENS
        elif isinstance(e, AttnRow):
            kinds[i] = TAG_ATTN_ROW
            row[i] = len(layers)
            p = np.asarray(e.probs, F32).reshape(-1)
            layers.append(int(e.layer))
            sizes.append(p.size)
            chunks.append(p)
        elif isinstance(e, SaddleTruth):
            kinds[i] = TAG_SADDLE_TRUTH
            truth[i] = np.asarray(e.ids).astype(np.int64)
        else:
            raise ValueError(f"unexpected trace event {e!r}")
    n = np.array(sizes, np.int64)
    off = np.zeros(len(sizes), np.int64)
    if len(sizes):
        off[1:] = np.cumsum(n)[:-1]
    payload = np.concatenate(chunks) if chunks else np.zeros(0, F32)
    return TraceIndex(header=header, kind=kinds, row=row, round_info=info, row_layer=np.array(layers, np.int64),
                      row_off=off, row_n=n.astype(np.int32), payload=payload, truth=truth)
