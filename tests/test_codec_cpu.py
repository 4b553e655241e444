"""Exponent-Huffman codec, host side (libxpgb C++ encoder): bit-exact with the reference."""

import hashlib

import numpy as np
import pytest

import paper_2604_02715_b200 as X
from paper_2604_02715_b200 import exponent_codec as XC
from paper_2604_02715_b200.errors import EmptyHistogramError, OddLengthError, SymbolNotInTableError, TruncatedStreamError


def _bf16(vals):
    return X.float32_to_bf16(np.asarray(vals, np.float32)).astype("<u2").tobytes()


def test_histogram_bins_and_odd_length():
    assert XC.build_histogram(_bf16([0.0] * 1000)).counts[0] == 1000
    assert XC.build_histogram(_bf16([1.0] * 8)).counts[127] == 8
    with pytest.raises(OddLengthError):
        XC.build_histogram(b"\x00\x01\x02")


@pytest.mark.parametrize("key", ["xpgc_2_2_16_32_6", "xpgc_3_2_32_64_4", "xpgc_4_8_256_512_7"])
def test_xpgc_bytes_identical_to_reference(golden, key):
    arrays, meta = golden
    _, N, L, H, F, seed = key.split("_")
    spec = X.ModelSpec(int(N), int(L), int(H), int(F))
    container = X.generate_synthetic_model(spec, int(seed), pin=False)
    cm = XC.CompressedModel.from_container(container, pin=False)
    np.testing.assert_array_equal(np.array(cm.table.code_lengths, np.uint8), arrays[key + "_lengths"])
    np.testing.assert_array_equal(cm.bits_lens.astype(np.int64), arrays[key + "_bits"])
    np.testing.assert_array_equal(cm.bit_counts.astype(np.int64), arrays[key + "_bitcount"])
    assert hashlib.sha256(cm.to_bytes()).hexdigest() == meta["cases"][key]["sha256"]
    assert cm.ratio == pytest.approx(meta["cases"][key]["ratio"])
    assert cm.ratio <= 0.85


def test_adversarial_and_random_streams(golden):
    arrays, meta = golden
    adv = np.arange(65536, dtype=np.uint16).astype("<u2").tobytes()
    t = XC.build_table(XC.build_histogram(adv))
    np.testing.assert_array_equal(np.array(t.code_lengths, np.uint8), arrays["codec_adv_lengths"])
    ct = XC.compress(adv, t)
    assert hashlib.sha256(ct.exponent_bitstream).hexdigest() == meta["cases"]["codec_adv"]["stream_sha256"]
    assert ct.exponent_bit_count == meta["cases"]["codec_adv"]["bit_count"]
    rnd = np.random.default_rng(9).integers(0, 65536, 200_000, dtype=np.uint16).astype("<u2").tobytes()
    t = XC.build_table(XC.build_histogram(rnd))
    np.testing.assert_array_equal(np.array(t.code_lengths, np.uint8), arrays["codec_rnd_lengths"])
    ct = XC.compress(rnd, t)
    assert hashlib.sha256(ct.exponent_bitstream).hexdigest() == meta["cases"]["codec_rnd"]["stream_sha256"]
    assert ct.effective_bits_per_value() >= 15.9


def test_length_cap_matches_reference(golden):
    arrays, _ = golden
    hist = XC.ExponentHistogram(tuple(int(v) for v in arrays["codec_skew_counts"]))
    t = XC.build_table(hist)
    np.testing.assert_array_equal(np.array(t.code_lengths, np.uint8), arrays["codec_skew_lengths"])
    assert max(t.code_lengths) <= 32


def test_table_edge_cases():
    t = XC.build_table(XC.ExponentHistogram(tuple(1 if i == 42 else 0 for i in range(256))))
    assert t.code_lengths[42] == 1 and sum(t.code_lengths) == 1
    with pytest.raises(EmptyHistogramError):
        XC.build_table(XC.ExponentHistogram((0,) * 256))
    with pytest.raises(SymbolNotInTableError):
        XC.compress(_bf16([2.0] * 4), XC.build_table(XC.build_histogram(_bf16([1.0] * 4))))


def test_chunk_index_rebuild_and_truncation():
    data = _bf16(np.random.default_rng(1).standard_normal(50_000) * 0.02)
    t = XC.build_table(XC.build_histogram(data))
    ct = XC.compress(data, t, chunk=256)
    from dataclasses import replace

    rec = XC._record(replace(ct, chunk_index=b""), t)  # index rebuilt by the host scan
    n = ct.value_count
    sm16 = (n + 15) & ~15
    bits16 = (len(ct.exponent_bitstream) + 8 + 15) & ~15
    nidx = (n + 255) // 256
    assert rec[sm16 + bits16:sm16 + bits16 + 4 * nidx].tobytes() == ct.chunk_index
    cut = replace(ct, exponent_bitstream=ct.exponent_bitstream[: len(ct.exponent_bitstream) // 4], chunk_index=b"")
    with pytest.raises(TruncatedStreamError):
        XC._record(cut, t)


def test_compressed_pool_layer_kind_order():
    """Records of one (layer, kind) are contiguous in the packed pool, experts ascending."""
    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    spec = X.ModelSpec(2, 5, 64, 128)
    cm = CompressedModel.from_container(X.generate_synthetic_model(spec, 1), pin=False)
    ids = list(X.iter_tensor_ids(spec))
    order = sorted(range(len(ids)), key=lambda i: (ids[i].layer, int(ids[i].kind), ids[i].expert))
    offs = [int(cm.rec_offsets[i]) for i in order]
    assert offs == sorted(offs) and offs[0] == 0
