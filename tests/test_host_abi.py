"""Host-side logic of the product behind the C ABI, on CPU: the library
loads and exports every symbol include/q8p.h declares; QSHP v1 reader/writer
is byte-compatible with the reference; tables, planner and bases equal the
oracle's; malformed artifacts raise the reference's typed errors
(test_pipeline.cpp:200-236).  No compute calls (no GPU here)."""
import os
import re
import struct

import numpy as np
import pytest

import paper_2402_04396_b200 as q8p
from conftest import ROOT, golden_names, load_case


def header_symbols():
    with open(os.path.join(ROOT, "include", "q8p.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(q8p_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = q8p.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), f"libq8p.so does not export {s}"
    assert set(syms) == set(q8p._SIGNATURES), "Python binding out of sync with include/q8p.h"
    assert q8p.lib().q8p_version().startswith(b"q8p")


def test_plan_hadamard_matches_reference_plans(kat, oracle):
    for n, pq in kat["plans"].items():
        assert list(q8p.plan_hadamard(int(n))) == pq
    assert q8p.plan_hadamard(11008) == (64, 172)
    assert q8p.plan_hadamard(28672) == (1024, 28)
    for bad in (0, 7, 36):
        with pytest.raises(q8p.SizeError):
            q8p.plan_hadamard(bad)
    for n in range(1, 2000):
        try:
            want = oracle.plan_hadamard(n)
        except Exception:
            with pytest.raises(q8p.SizeError):
                q8p.plan_hadamard(n)
            continue
        assert q8p.plan_hadamard(n) == want


def test_hadamard_bases_match_oracle(oracle):
    for q in (1, 4, 12, 20, 28, 172):
        assert np.array_equal(q8p.hadamard_base(q), oracle.hadamard_base(q))
    with pytest.raises(q8p.SizeError):
        q8p.hadamard_base(9)


def test_codebook_tables_match_oracle(oracle):
    d, p = q8p.codebook_table(q8p.CB_E8P_2BIT)
    od, op = oracle.e8p_tables()
    assert np.array_equal(d, od) and np.array_equal(p, op)
    e, _ = q8p.codebook_table(q8p.CB_E8_1BIT)
    assert np.array_equal(e.astype(np.float64) / 2, oracle.e8_1bit_table())


def test_host_decode_all_words_bit_exact(oracle):
    want = oracle.e8p_decode_all()
    got = np.stack([q8p.e8p_decode_host(w) for w in range(65536)]).astype(np.float64)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name", golden_names())
def test_qshp_roundtrip_byte_identical(name):
    art, _, _ = load_case(name)
    assert q8p.reserialize(art) == art
    info = q8p.inspect_artifact(art)
    assert info["serialized_size"] == len(art)


def test_qshp_size_arithmetic():
    # test_pipeline.cpp:83-84: 32x32 2-bit rht = 16 + 13 + 8 + 32*4*2 = 293 bytes
    m = n = 32
    body = b"QSHP" + struct.pack("<HIIBB", 1, m, n, 0, 1) + bytes([8]) + b"e8p-2bit" + struct.pack("<f", 1.0)
    art = body + bytes(4) + bytes(4) + bytes(m * n // 8 * 2)
    assert len(art) == 293
    assert q8p.inspect_artifact(art)["serialized_size"] == 293
    assert q8p.reserialize(art) == art


def test_malformed_artifacts_raise_typed_errors():
    art, _, _ = load_case("e8p2_64x64")
    bad = bytearray(art); bad[0] = ord("X")
    with pytest.raises(q8p.BadMagicError):
        q8p.inspect_artifact(bytes(bad))
    bad = bytearray(art); bad[4] = 2
    with pytest.raises(q8p.UnsupportedVersionError):
        q8p.inspect_artifact(bytes(bad))
    for cut in (3, len(art) - 1, 10):
        with pytest.raises(q8p.TruncatedArtifactError):
            q8p.inspect_artifact(art[:cut])
    with pytest.raises(q8p.FormatError):
        q8p.inspect_artifact(art + b"\0")
    bad = bytearray(art); bad[14] = 9
    with pytest.raises(q8p.FormatError):
        q8p.inspect_artifact(bytes(bad))
    bad = bytearray(art); bad[17] = ord("x")
    with pytest.raises(q8p.ValidationError):
        q8p.inspect_artifact(bytes(bad))


def test_sign_pad_bits_masked_on_roundtrip():
    # bitpack.cpp:16-26: from_bytes zeroes pad bits -> reserialize normalizes them.
    m, n = 12, 16
    body = b"QSHP" + struct.pack("<HIIBB", 1, m, n, 0, 1) + bytes([8]) + b"e8p-2bit" + struct.pack("<f", 0.5)
    art = body + bytes([0xFF, 0xFF]) + bytes([0x00, 0x00]) + bytes(m * n // 8 * 2)
    out = q8p.reserialize(art)
    assert out[len(body):len(body) + 2] == bytes([0xFF, 0x0F])


def test_compute_calls_fail_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present: covered by -m gpu tests")
    except ImportError:
        pass
    art, _, _ = load_case("e8p2_64x64")
    with pytest.raises(q8p.DeviceError):
        q8p.Layer.from_qshp(art)
