"""Lossless exponent-Huffman codec for bf16 expert weights (reference xpg codec.py:1-475).

Only the 8 exponent bits are entropy-coded with one canonical Huffman table per
model; sign + mantissa travel raw, one byte per value.  The stream bytes this
module produces are bit-identical to the reference's ``compress``; XPGC
containers are byte-identical.

B200 split of the work:

* encoding (``compress``, ``CompressedModel.from_container``) runs in libxpgb's
  multi-threaded C++ encoder on the host — it happens once per model;
* decoding (``decompress``, and every compressed page-in of the paged runner)
  runs on the GPU (``k_exp_decode``): a per-chunk bit index, kept as side
  metadata next to the reference stream, lets thousands of threads decode one
  tensor in parallel straight into a ring block.
"""

from __future__ import annotations

import ctypes as C
import heapq
import os
import struct
import zlib
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from ._lib import call, lib
from .errors import (
    ContainerFormatError,
    EmptyHistogramError,
    OddLengthError,
    SymbolNotInTableError,
    TruncatedStreamError,
)
from .geometry import XPGW_VERSION, ModelSpec, TensorKind, WeightContainer, iter_tensor_ids

XPGC_MAGIC = b"XPGC"
_XPGC_HEADER = struct.Struct("<4sIQQQQ")
_RECORD = struct.Struct("<QQ")
TENSOR_HEADER_BYTES = _RECORD.size
NUM_SYMBOLS = 256
MAX_CODE_LENGTH = 32
DEFAULT_CHUNK = 256  # values per decode thread: 1509 GB/s vs 962 at 1024 (Mixtral gate/up, B200)


def chunk_for(spec: ModelSpec) -> int:
    """Decode chunk for a model's tensors: 256 values for big tensors (Mixtral's 117M-value
    gate/up: 1,509 GB/s vs 1,462 at 128), 128 for smaller ones, where more threads per tensor
    pay for the doubled chunk index (DSv3's 14.7M values: 908 vs 717 GB/s; Qwen3's 3.1M:
    265 vs 158)."""
    return 256 if spec.value_count(TensorKind.GATE_UP) >= (32 << 20) else 128
_THREADS = max(1, os.cpu_count() or 1)


def _u8p(arr):
    return arr.ctypes.data_as(C.POINTER(C.c_uint8))


def _as_words(data) -> np.ndarray:
    if isinstance(data, np.ndarray):
        raw = np.ascontiguousarray(data).reshape(-1).view(np.uint8)
    else:
        raw = np.frombuffer(bytes(data) if not isinstance(data, (bytes, bytearray, memoryview)) else data,
                            dtype=np.uint8)
    if raw.size % 2:
        raise OddLengthError(f"bf16 payload has odd length {raw.size}")
    return raw.view("<u2")


def exponent_bytes(data) -> np.ndarray:
    return ((_as_words(data) >> 7) & 0xFF).astype(np.uint8)


def sign_mantissa_bytes(data) -> np.ndarray:
    w = _as_words(data)
    return (((w >> 8) & 0x80) | (w & 0x7F)).astype(np.uint8)


@dataclass(frozen=True)
class ExponentHistogram:
    counts: tuple

    def __post_init__(self):
        if len(self.counts) != NUM_SYMBOLS:
            raise ValueError("histogram needs exactly 256 bins")

    @property
    def total(self) -> int:
        return sum(self.counts)

    def entropy_bits(self) -> float:
        c = np.asarray(self.counts, dtype=np.float64)
        t = c.sum()
        if t == 0:
            return 0.0
        p = c[c > 0] / t
        return float(-(p * np.log2(p)).sum())


def build_histogram(data) -> ExponentHistogram:
    words = _as_words(data)
    counts = (C.c_uint64 * NUM_SYMBOLS)()
    call("xpgb_codec_histogram", C.c_void_p(words.ctypes.data), C.c_uint64(words.nbytes), counts, _THREADS)
    return ExponentHistogram(tuple(int(v) for v in counts))


def _optimal_lengths(counts) -> list:
    """Huffman code lengths with the reference's deterministic tie-breaking
    (codec.py:92-119): leaves (count, symbol), merged nodes (count, 256 + merge index)."""
    nodes = [(c, s, None) for s, c in enumerate(counts) if c > 0]
    if not nodes:
        raise EmptyHistogramError("cannot build a table from an empty histogram")
    lengths = [0] * NUM_SYMBOLS
    if len(nodes) == 1:
        lengths[nodes[0][1]] = 1
        return lengths
    heapq.heapify(nodes)
    serial = NUM_SYMBOLS
    while len(nodes) > 1:
        lo = heapq.heappop(nodes)
        hi = heapq.heappop(nodes)
        heapq.heappush(nodes, (lo[0] + hi[0], serial, (lo, hi)))
        serial += 1
    todo = [(nodes[0], 0)]
    while todo:
        (_, sym, kids), depth = todo.pop()
        if kids is None:
            lengths[sym] = depth
        else:
            todo.extend(((kids[0], depth + 1), (kids[1], depth + 1)))
    return lengths


def _cap_lengths(lengths: list, cap: int) -> list:
    """Clamp lengths to `cap`, then lengthen the deepest cheap codes until Kraft holds
    (codec.py:122-142)."""
    if max(lengths) <= cap:
        return lengths
    out = [min(v, cap) if v else 0 for v in lengths]
    budget = 1 << cap
    kraft = sum(1 << (cap - v) for v in out if v)
    while kraft > budget:
        for v in range(cap - 1, 0, -1):
            hit = next((s for s, ln in enumerate(out) if ln == v), None)
            if hit is not None:
                out[hit] += 1
                kraft -= 1 << (cap - v - 1)
                break
    return out


@dataclass(frozen=True)
class HuffmanTable:
    code_lengths: tuple
    codes: tuple = field(repr=False, default=())

    @classmethod
    def from_lengths(cls, lengths) -> "HuffmanTable":
        lengths = tuple(int(v) for v in lengths)
        if len(lengths) != NUM_SYMBOLS:
            raise ValueError("need exactly 256 code lengths")
        if any(v < 0 or v > MAX_CODE_LENGTH for v in lengths):
            raise ValueError(f"code lengths must lie in [0, {MAX_CODE_LENGTH}]")
        present = sorted((v, s) for s, v in enumerate(lengths) if v)
        if not present:
            raise EmptyHistogramError("table has no symbols")
        if sum(2.0 ** -v for v, _ in present) > 1.0 + 1e-12:
            raise ValueError("code lengths violate the Kraft inequality")
        codes = [0] * NUM_SYMBOLS
        code, prev = 0, 0
        for v, s in present:
            code <<= v - prev
            codes[s] = code
            code += 1
            prev = v
        return cls(code_lengths=lengths, codes=tuple(codes))

    @property
    def table_id(self) -> int:
        return zlib.crc32(bytes(self.code_lengths))

    def lengths_array(self) -> np.ndarray:
        return np.asarray(self.code_lengths, dtype=np.uint8)

    def expected_bits(self, hist: ExponentHistogram) -> float:
        t = hist.total
        return sum(c * self.code_lengths[s] for s, c in enumerate(hist.counts) if c) / t if t else 0.0


def build_table(hist: ExponentHistogram) -> HuffmanTable:
    if hist.total < 1:
        raise EmptyHistogramError("histogram is empty")
    return HuffmanTable.from_lengths(_cap_lengths(_optimal_lengths(hist.counts), MAX_CODE_LENGTH))


@dataclass(frozen=True)
class CompressedTensor:
    value_count: int
    sign_mantissa_plane: bytes
    exponent_bitstream: bytes
    exponent_bit_count: int
    table_id: int
    tensor_id: object = None
    chunk_index: bytes = field(default=b"", repr=False)  # B200 side metadata (u32 per chunk)
    chunk: int = DEFAULT_CHUNK

    @property
    def compressed_bytes(self) -> int:
        return TENSOR_HEADER_BYTES + self.value_count + len(self.exponent_bitstream)

    def effective_bits_per_value(self) -> float:
        if self.value_count < 1:
            raise ValueError("effective bits undefined for an empty tensor")
        return 8.0 + self.exponent_bit_count / self.value_count


def compress(data, table: HuffmanTable, tensor_id=None, chunk: int = DEFAULT_CHUNK) -> CompressedTensor:
    words = _as_words(data)
    n = words.size
    lengths = table.lengths_array()
    sm = np.zeros(max(n, 1), dtype=np.uint8)
    cap = max(1, (n * int(lengths.max()) + 7) // 8)
    bits = np.zeros(cap, dtype=np.uint8)
    index = np.zeros(max(1, (n + chunk - 1) // chunk), dtype=np.uint32)
    blen, bcount = C.c_uint64(), C.c_uint64()
    call("xpgb_codec_encode", C.c_void_p(words.ctypes.data), C.c_uint64(words.nbytes), _u8p(lengths),
         C.c_void_p(sm.ctypes.data), C.c_void_p(bits.ctypes.data), C.c_uint64(cap), C.byref(blen), C.byref(bcount),
         index.ctypes.data_as(C.POINTER(C.c_uint32)), chunk)
    nidx = (n + chunk - 1) // chunk
    return CompressedTensor(n, sm[:n].tobytes(), bits[:blen.value].tobytes(), int(bcount.value), table.table_id,
                            tensor_id, index[:nidx].tobytes(), chunk)


def _stream_bits(ct: CompressedTensor, table: HuffmanTable) -> int:
    """Exact exponent bit count of a stream (host scan; XPGC does not store it)."""
    if ct.exponent_bit_count or not ct.value_count:
        return int(ct.exponent_bit_count)
    nb = len(ct.exponent_bitstream)
    bits = np.frombuffer(ct.exponent_bitstream, dtype=np.uint8) if nb else np.zeros(1, np.uint8)
    used = C.c_uint64()
    call("xpgb_codec_index", C.c_void_p(bits.ctypes.data), C.c_uint64(nb), C.c_uint64(ct.value_count),
         _u8p(table.lengths_array()), ct.chunk, None, C.byref(used))
    return int(used.value)


def _record(ct: CompressedTensor, table: HuffmanTable) -> np.ndarray:
    """Packed record (sm | stream + 8 pad | index), 16-byte aligned parts."""
    n, nb, ch = ct.value_count, len(ct.exponent_bitstream), ct.chunk
    index = ct.chunk_index
    if len(index) != 4 * ((n + ch - 1) // ch):
        idx = np.zeros(max(1, (n + ch - 1) // ch), dtype=np.uint32)
        bits = np.frombuffer(ct.exponent_bitstream, dtype=np.uint8) if nb else np.zeros(1, np.uint8)
        call("xpgb_codec_index", C.c_void_p(bits.ctypes.data), C.c_uint64(nb), C.c_uint64(n),
             _u8p(table.lengths_array()), ch, idx.ctypes.data_as(C.POINTER(C.c_uint32)), None)
        index = idx[:(n + ch - 1) // ch].tobytes()
    size = int(lib().xpgb_codec_record_bytes(n, nb, ch))
    rec = np.zeros(size, dtype=np.uint8)
    sm16 = (n + 15) & ~15
    bits16 = (nb + 8 + 15) & ~15
    rec[:n] = np.frombuffer(ct.sign_mantissa_plane, dtype=np.uint8)
    rec[sm16:sm16 + nb] = np.frombuffer(ct.exponent_bitstream, dtype=np.uint8)
    rec[sm16 + bits16:sm16 + bits16 + len(index)] = np.frombuffer(index, dtype=np.uint8)
    return rec


def decompress(ct: CompressedTensor, table: HuffmanTable, device: int = 0) -> bytes:
    """GPU decode of one tensor (bit-exact, NaN/Inf/subnormals included)."""
    if ct.table_id != table.table_id:
        raise SymbolNotInTableError(f"tensor was coded with table {ct.table_id:#x}, got {table.table_id:#x}")
    n = ct.value_count
    if len(ct.sign_mantissa_plane) != n:
        raise ContainerFormatError(f"sign/mantissa plane is {len(ct.sign_mantissa_plane)} bytes for {n} values")
    if n == 0:
        return b""
    if ct.exponent_bit_count and len(ct.exponent_bitstream) < (ct.exponent_bit_count + 7) // 8:
        raise TruncatedStreamError(f"bitstream ended before all {n} values", byte_offset=len(ct.exponent_bitstream),
                                   tensor_id=ct.tensor_id)
    rec = _record(ct, table)  # validates the stream (TruncatedStreamError / InvalidCodeError) when indexing
    import torch

    from .device import _torch, current_stream_ptr

    _torch()
    d_rec = torch.from_numpy(rec).to(f"cuda:{device}")
    out = torch.empty(n, dtype=torch.int16, device=f"cuda:{device}")
    call("xpgb_codec_decode", C.c_void_p(d_rec.data_ptr()), C.c_uint64(n), C.c_uint64(len(ct.exponent_bitstream)),
         ct.chunk, _u8p(table.lengths_array()), C.c_void_p(out.data_ptr()), C.c_void_p(current_stream_ptr(device)))
    return out.cpu().numpy().view("<u2").tobytes()


def optimal_code_cost_bits(hist: ExponentHistogram) -> int:
    counts = [c for c in hist.counts if c > 0]
    if not counts:
        raise EmptyHistogramError("histogram is empty")
    if len(counts) == 1:
        return counts[0]
    heapq.heapify(counts)
    total = 0
    while len(counts) > 1:
        m = heapq.heappop(counts) + heapq.heappop(counts)
        total += m
        heapq.heappush(counts, m)
    return total


class CompressedModel:
    """Whole model under one exponent table, packed for the GPU page-in path.

    ``pool`` holds every tensor's packed record (container order) in one
    buffer — pinned when a GPU is present — that the runner DMAs from.
    """

    def __init__(self, spec: ModelSpec, table: HuffmanTable, pool, rec_offsets, bits_lens, bit_counts,
                 chunk: int = DEFAULT_CHUNK):
        self.spec = spec
        self.table = table
        self.pool = pool                      # uint8 torch tensor (pinned) or numpy array
        self.rec_offsets = np.asarray(rec_offsets, dtype=np.uint64)
        self.bits_lens = np.asarray(bits_lens, dtype=np.uint64)
        self.bit_counts = np.asarray(bit_counts, dtype=np.uint64)
        self.chunk = chunk
        self._ids = list(iter_tensor_ids(spec))
        self._slot = {tid: i for i, tid in enumerate(self._ids)}

    @classmethod
    def from_container(cls, container: WeightContainer, chunk: int | None = None, pin: bool = True):
        spec = container.spec
        table = build_table(build_histogram(container.words))
        return cls.pack(container.words, spec, table, chunk=chunk or chunk_for(spec), pin=pin)

    @classmethod
    def pack(cls, words: np.ndarray, spec: ModelSpec, table: HuffmanTable, chunk: int = DEFAULT_CHUNK,
             pin: bool = True, n_layers: int | None = None, experts: int | None = None):
        from .geometry import _pinned_bytes

        ids = list(iter_tensor_ids(spec))
        counts = np.array([spec.value_count(t.kind) for t in ids], dtype=np.uint64)
        nt = len(ids)
        offs = np.zeros(nt, dtype=np.uint64)
        blens = np.zeros(nt, dtype=np.uint64)
        bcnt = np.zeros(nt, dtype=np.uint64)
        total = C.c_uint64()
        lengths = table.lengths_array()
        p64 = C.POINTER(C.c_uint64)
        # records in (layer, kind, expert) order: a layer's records of one kind are contiguous,
        # so the page-in stages runs of small records with one copy (offsets stay per tensor id)
        order = np.array(sorted(range(nt), key=lambda i: (ids[i].layer, int(ids[i].kind), ids[i].expert)),
                         dtype=np.int32)
        args = (C.c_void_p(words.ctypes.data), nt, counts.ctypes.data_as(p64), _u8p(lengths), chunk, _THREADS,
                order.ctypes.data_as(C.POINTER(C.c_int32)))
        call("xpgb_codec_pack", *args, None, C.c_uint64(0), C.byref(total), offs.ctypes.data_as(p64),
             blens.ctypes.data_as(p64), bcnt.ctypes.data_as(p64))
        pool = _pinned_bytes(int(total.value), pin)
        call("xpgb_codec_pack", *args, C.c_void_p(pool.data_ptr()), C.c_uint64(pool.numel()), C.byref(total),
             offs.ctypes.data_as(p64), blens.ctypes.data_as(p64), bcnt.ctypes.data_as(p64))
        return cls(spec, table, pool, offs, blens, bcnt, chunk)

    # ---- per-tensor views (reference-compatible)
    def _rec(self, i: int) -> np.ndarray:
        n = self.spec.value_count(self._ids[i].kind)
        size = int(lib().xpgb_codec_record_bytes(n, int(self.bits_lens[i]), self.chunk))
        arr = self.pool.numpy() if hasattr(self.pool, "numpy") else self.pool
        off = int(self.rec_offsets[i])
        return arr[off:off + size]

    def compressed_tensor(self, tid) -> CompressedTensor:
        i = self._slot[tid]
        n = self.spec.value_count(tid.kind)
        rec = self._rec(i)
        nb = int(self.bits_lens[i])
        sm16 = (n + 15) & ~15
        bits16 = (nb + 8 + 15) & ~15
        nidx = (n + self.chunk - 1) // self.chunk
        return CompressedTensor(n, rec[:n].tobytes(), rec[sm16:sm16 + nb].tobytes(), int(self.bit_counts[i]),
                                self.table.table_id, tid, rec[sm16 + bits16:sm16 + bits16 + 4 * nidx].tobytes(),
                                self.chunk)

    @property
    def tensors(self) -> dict:
        return {tid: self.compressed_tensor(tid) for tid in self._ids}

    def tensor_bytes(self, tid) -> bytes:
        return decompress(self.compressed_tensor(tid), self.table)

    @property
    def compressed_payload_bytes(self) -> int:
        n = np.array([self.spec.value_count(t.kind) for t in self._ids], dtype=np.uint64)
        return int((TENSOR_HEADER_BYTES + n + self.bits_lens).sum())

    @property
    def ratio(self) -> float:
        return self.compressed_payload_bytes / self.spec.total_bytes

    @property
    def wire_bytes(self) -> int:
        """Bytes the GPU page-in actually moves (records incl. chunk index and alignment)."""
        arr = self.pool.numel() if hasattr(self.pool, "numel") else self.pool.size
        return int(arr)

    def to_bytes(self) -> bytes:
        s = self.spec
        parts = [_XPGC_HEADER.pack(XPGC_MAGIC, XPGW_VERSION, s.num_layers, s.experts_per_layer, s.hidden_dim,
                                   s.intermediate_dim), bytes(self.table.code_lengths)]
        for i, tid in enumerate(self._ids):
            n = s.value_count(tid.kind)
            nb = int(self.bits_lens[i])
            rec = self._rec(i)
            sm16 = (n + 15) & ~15
            parts += [_RECORD.pack(n, nb), rec[:n].tobytes(), rec[sm16:sm16 + nb].tobytes()]
        return b"".join(parts)

    @classmethod
    def from_bytes(cls, raw: bytes, chunk: int | None = None) -> "CompressedModel":
        if len(raw) < _XPGC_HEADER.size:
            raise ContainerFormatError("compressed container shorter than header")
        magic, version, n, l, h, f = _XPGC_HEADER.unpack_from(raw, 0)
        if magic != XPGC_MAGIC:
            raise ContainerFormatError(f"bad magic {magic!r}, expected {XPGC_MAGIC!r}")
        if version != XPGW_VERSION:
            raise ContainerFormatError(f"unsupported container version {version}")
        spec = ModelSpec(n, l, h, f)
        chunk = chunk or chunk_for(spec)
        pos = _XPGC_HEADER.size
        if len(raw) < pos + NUM_SYMBOLS:
            raise ContainerFormatError("compressed container truncated in code lengths")
        table = HuffmanTable.from_lengths(raw[pos:pos + NUM_SYMBOLS])
        pos += NUM_SYMBOLS
        cts = []
        for tid in iter_tensor_ids(spec):
            if len(raw) < pos + TENSOR_HEADER_BYTES:
                raise TruncatedStreamError(f"record header for {tid} truncated", byte_offset=pos, tensor_id=tid)
            cnt, slen = _RECORD.unpack_from(raw, pos)
            pos += TENSOR_HEADER_BYTES
            if cnt != spec.value_count(tid.kind):
                raise ContainerFormatError(f"{tid}: value count {cnt} does not match geometry")
            end = pos + cnt + slen
            if len(raw) < end:
                raise TruncatedStreamError(f"payload for {tid} truncated", byte_offset=pos, tensor_id=tid)
            cts.append(CompressedTensor(cnt, raw[pos:pos + cnt], raw[pos + cnt:end], 0, table.table_id, tid,
                                        b"", chunk))
            pos = end
        return cls.from_tensors(spec, table, cts, chunk)

    @classmethod
    def from_tensors(cls, spec: ModelSpec, table: HuffmanTable, cts, chunk: int = DEFAULT_CHUNK):
        recs = [_record(ct, table) for ct in cts]
        offs = np.zeros(len(recs), dtype=np.uint64)
        at = 0
        for i, r in enumerate(recs):
            offs[i] = at
            at += r.size
        from .geometry import _pinned_bytes

        pool = _pinned_bytes(at, True)
        arr = pool.numpy()
        for i, r in enumerate(recs):
            arr[int(offs[i]):int(offs[i]) + r.size] = r
        lengths = table.code_lengths
        bit_counts = [_stream_bits(ct, table) for ct in cts]
        return cls(spec, table, pool, offs, [len(ct.exponent_bitstream) for ct in cts], bit_counts, chunk)

    def write(self, path) -> None:
        Path(path).write_bytes(self.to_bytes())

    @classmethod
    def read(cls, path) -> "CompressedModel":
        return cls.from_bytes(Path(path).read_bytes())
