"""ctypes bindings for the two CPU oracles.  TEST INFRASTRUCTURE ONLY
(imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg; never by the product package).

  Ref     -> oracle/_ref/libref_latq.so: the UNMODIFIED reference latq sources
             compiled in place (oracle/Makefile `ref`), plus ref_glue.cpp.
  Oracle  -> oracle/build/liblatq_oracle.so: the C restatement latq_oracle.c
             (bit-identical to Ref on every shape Ref can plan; also plans
             n = 11008 via the order-172 base).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libref_latq.so")
ORACLE_SO = os.path.join(HERE, "build", "liblatq_oracle.so")

_P = ctypes.c_void_p


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class Ref:
    """The reference library itself (compiled from /root/reference sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build with `make -C oracle ref` (needs /root/reference)")
        L = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_substream_seed.restype = ctypes.c_uint64
        L.ref_substream_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.ref_quantize_hi.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                      ctypes.c_int,
                                      ctypes.POINTER(ctypes.POINTER(ctypes.c_uint8)), ctypes.POINTER(ctypes.c_size_t)]
        L.ref_quantize_layer.argtypes = [_P, _P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_uint64, ctypes.c_int,
                                         ctypes.POINTER(ctypes.POINTER(ctypes.c_uint8)), ctypes.POINTER(ctypes.c_size_t)]
        L.ref_roundtrip.argtypes = [ctypes.c_char_p, ctypes.c_size_t,
                                    ctypes.POINTER(ctypes.POINTER(ctypes.c_uint8)), ctypes.POINTER(ctypes.c_size_t)]
        L.ref_infer.argtypes = [ctypes.c_char_p, ctypes.c_size_t, _P, ctypes.c_int, _P, ctypes.c_int]
        L.ref_dequantize.argtypes = [ctypes.c_char_p, ctypes.c_size_t, _P]
        L.ref_decode_stage.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, _P]
        L.ref_e8p_decode.argtypes = [ctypes.c_uint16, _P]
        L.ref_e8p_encode.argtypes = [_P, ctypes.POINTER(ctypes.c_uint16)]
        L.ref_e8p_tables.argtypes = [_P, _P]
        L.ref_codebook_decode.argtypes = [ctypes.c_char_p, ctypes.c_uint32, _P, ctypes.POINTER(ctypes.c_int)]
        L.ref_plan_hadamard.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]
        L.ref_hadamard_base.argtypes = [ctypes.c_size_t, _P]
        L.ref_had_apply.argtypes = [ctypes.c_size_t, _P, ctypes.c_int]
        L.ref_side_apply.argtypes = [ctypes.c_size_t, _P, _P, ctypes.c_int]
        L.ref_gen_weights.argtypes = [ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64, _P]
        L.ref_random_signs.argtypes = [ctypes.c_size_t, ctypes.c_uint64, _P]
        L.ref_rfft_apply.argtypes = [ctypes.c_size_t, _P, _P, ctypes.c_int]
        L.ref_rvq_quantize.argtypes = [ctypes.c_int, _P, _P, ctypes.c_size_t, _P]
        L.ref_random_phases.argtypes = [ctypes.c_size_t, ctypes.c_uint64, _P]
        L.ref_artifact_info.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint32),
                                        ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int)]
        self.L = L

    def _ck(self, st: int) -> None:
        if st != 0:
            raise OracleError(st, self.L.ref_last_error().decode())

    def _bytes_out(self, fn, *args) -> bytes:
        out = ctypes.POINTER(ctypes.c_uint8)()
        n = ctypes.c_size_t()
        self._ck(fn(*args, ctypes.byref(out), ctypes.byref(n)))
        b = ctypes.string_at(out, n.value)
        self.L.ref_free(out)
        return b

    def substream_seed(self, seed: int, stream: int) -> int:
        return int(self.L.ref_substream_seed(seed, stream))

    def quantize_hi(self, m: int, n: int, bits: int, seed: int, threads: int = 8, transform: int = 0) -> bytes:
        """transform 0 = rht, 1 = rfft (TransformKind)."""
        return self._bytes_out(self.L.ref_quantize_hi, m, n, bits, transform, seed, threads)

    def quantize_layer(self, w: np.ndarray, h: np.ndarray | None, bits: int, seed: int, threads: int = 8,
                       transform: int = 0) -> bytes:
        w = np.ascontiguousarray(w, dtype=np.float64)
        hp = None if h is None else _ptr(np.ascontiguousarray(h, dtype=np.float64))
        m, n = w.shape
        return self._bytes_out(self.L.ref_quantize_layer, _ptr(w), hp, m, n, bits, transform, seed, threads)

    def roundtrip(self, data: bytes) -> bytes:
        return self._bytes_out(self.L.ref_roundtrip, data, len(data))

    def artifact_info(self, data: bytes) -> tuple[int, int, int]:
        m, n, s = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_int()
        self._ck(self.L.ref_artifact_info(data, len(data), ctypes.byref(m), ctypes.byref(n), ctypes.byref(s)))
        return m.value, n.value, s.value

    def infer(self, data: bytes, x: np.ndarray, threads: int = 1) -> np.ndarray:
        m, n, _ = self.artifact_info(data)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, n)
        y = np.zeros((x.shape[0], m))
        self._ck(self.L.ref_infer(data, len(data), _ptr(x), x.shape[0], _ptr(y), threads))
        return y

    def dequantize(self, data: bytes) -> np.ndarray:
        m, n, _ = self.artifact_info(data)
        w = np.zeros((m, n))
        self._ck(self.L.ref_dequantize(data, len(data), _ptr(w)))
        return w

    def decode_stage(self, data: bytes, stage: int) -> np.ndarray:
        m, n, _ = self.artifact_info(data)
        w = np.zeros((m, n))
        self._ck(self.L.ref_decode_stage(data, len(data), stage, _ptr(w)))
        return w

    def e8p_decode(self, word: int) -> np.ndarray:
        out = np.zeros(8)
        self._ck(self.L.ref_e8p_decode(word, _ptr(out)))
        return out

    def e8p_encode(self, v: np.ndarray) -> int:
        v = np.ascontiguousarray(v, dtype=np.float64)
        w = ctypes.c_uint16()
        self._ck(self.L.ref_e8p_encode(_ptr(v), ctypes.byref(w)))
        return w.value

    def e8p_tables(self) -> tuple[np.ndarray, np.ndarray]:
        d = np.zeros((256, 8), dtype=np.int8)
        p = np.zeros(256, dtype=np.uint8)
        self.L.ref_e8p_tables(_ptr(d), _ptr(p))
        return d, p

    def codebook_decode(self, cid: str, code: int) -> np.ndarray:
        out = np.zeros(8)
        dim = ctypes.c_int()
        self._ck(self.L.ref_codebook_decode(cid.encode(), code, _ptr(out), ctypes.byref(dim)))
        return out[: dim.value]

    def plan_hadamard(self, n: int) -> tuple[int, int]:
        p, q = ctypes.c_size_t(), ctypes.c_size_t()
        self._ck(self.L.ref_plan_hadamard(n, ctypes.byref(p), ctypes.byref(q)))
        return p.value, q.value

    def hadamard_base(self, q: int) -> np.ndarray:
        out = np.zeros(q * q, dtype=np.int8)
        self._ck(self.L.ref_hadamard_base(q, _ptr(out)))
        return out.reshape(q, q)

    def had_apply(self, x: np.ndarray, transpose: bool = False) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.float64).copy()
        self._ck(self.L.ref_had_apply(y.size, _ptr(y), int(transpose)))
        return y

    def side_apply(self, signs: np.ndarray, x: np.ndarray, transpose: bool = False) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.float64).copy()
        s = np.ascontiguousarray(signs, dtype=np.uint8)
        self._ck(self.L.ref_side_apply(y.size, _ptr(s), _ptr(y), int(transpose)))
        return y

    def gen_weights(self, m: int, n: int, seed: int) -> np.ndarray:
        w = np.zeros((m, n))
        self._ck(self.L.ref_gen_weights(m, n, seed, _ptr(w)))
        return w

    def rfft_apply(self, phases: np.ndarray, x: np.ndarray, transpose: bool = False) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.float64).copy()
        ph = np.ascontiguousarray(phases, dtype=np.float64)
        assert ph.size == y.size // 2
        self._ck(self.L.ref_rfft_apply(y.size, _ptr(ph), _ptr(y), int(transpose)))
        return y

    def rvq_quantize(self, bits: int, scales, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 8)
        sc = np.ascontiguousarray(scales, dtype=np.float64)
        out = np.zeros((sc.size, v.shape[0]), dtype=np.uint16)
        self._ck(self.L.ref_rvq_quantize(bits, _ptr(sc), _ptr(v), v.shape[0], _ptr(out)))
        return out

    def random_phases(self, n: int, seed: int) -> np.ndarray:
        out = np.zeros(n // 2)
        self._ck(self.L.ref_random_phases(n, seed, _ptr(out)))
        return out

    def random_signs(self, n: int, seed: int) -> np.ndarray:
        out = np.zeros((n + 7) // 8, dtype=np.uint8)
        self.L.ref_random_signs(n, seed, _ptr(out))
        return out


class Oracle:
    """The C restatement (oracle/latq_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build with `make -C oracle oracle`")
        L = ctypes.CDLL(path)
        L.oracle_e8p_tables.argtypes = [_P, _P]
        L.oracle_e8p_decode.argtypes = [ctypes.c_uint16, _P]
        L.oracle_e8p_decode.restype = None
        L.oracle_e8_1bit_table.argtypes = [_P]
        L.oracle_hadamard_base.argtypes = [ctypes.c_size_t, _P]
        L.oracle_plan_hadamard.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]
        L.oracle_had_apply.argtypes = [ctypes.c_size_t, _P, ctypes.c_int]
        L.oracle_side_apply.argtypes = [ctypes.c_size_t, _P, _P, ctypes.c_int]
        L.oracle_artifact_info.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint32),
                                           ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int)]
        L.oracle_infer.argtypes = [ctypes.c_char_p, ctypes.c_size_t, _P, ctypes.c_int, _P, ctypes.c_int]
        L.oracle_decode_stage.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, _P]
        L.oracle_rfft_apply.argtypes = [ctypes.c_size_t, _P, _P, ctypes.c_int]
        self.L = L

    @staticmethod
    def _ck(st: int) -> None:
        if st != 0:
            raise OracleError(st)

    def e8p_tables(self) -> tuple[np.ndarray, np.ndarray]:
        d = np.zeros((256, 8), dtype=np.int8)
        p = np.zeros(256, dtype=np.uint8)
        self._ck(self.L.oracle_e8p_tables(_ptr(d), _ptr(p)))
        return d, p

    def e8p_decode(self, word: int) -> np.ndarray:
        out = np.zeros(8)
        self.L.oracle_e8p_decode(word, _ptr(out))
        return out

    def e8p_decode_all(self) -> np.ndarray:
        out = np.zeros((65536, 8))
        for w in range(65536):
            self.L.oracle_e8p_decode(w, _ptr(out[w]))
        return out

    def e8_1bit_table(self) -> np.ndarray:
        out = np.zeros((256, 8))
        self._ck(self.L.oracle_e8_1bit_table(_ptr(out)))
        return out

    def plan_hadamard(self, n: int) -> tuple[int, int]:
        p, q = ctypes.c_size_t(), ctypes.c_size_t()
        self._ck(self.L.oracle_plan_hadamard(n, ctypes.byref(p), ctypes.byref(q)))
        return p.value, q.value

    def hadamard_base(self, q: int) -> np.ndarray:
        out = np.zeros(q * q, dtype=np.int8)
        self._ck(self.L.oracle_hadamard_base(q, _ptr(out)))
        return out.reshape(q, q)

    def had_apply(self, x: np.ndarray, transpose: bool = False) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.float64).copy()
        self._ck(self.L.oracle_had_apply(y.size, _ptr(y), int(transpose)))
        return y

    def side_apply(self, signs: np.ndarray, x: np.ndarray, transpose: bool = False) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.float64).copy()
        s = np.ascontiguousarray(signs, dtype=np.uint8)
        self._ck(self.L.oracle_side_apply(y.size, _ptr(s), _ptr(y), int(transpose)))
        return y

    def rfft_apply(self, phases: np.ndarray, x: np.ndarray, transpose: bool = False) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.float64).copy()
        ph = np.ascontiguousarray(phases, dtype=np.float64)
        assert ph.size == y.size // 2
        self._ck(self.L.oracle_rfft_apply(y.size, _ptr(ph), _ptr(y), int(transpose)))
        return y

    def artifact_info(self, data: bytes) -> tuple[int, int, int]:
        m, n, s = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_int()
        self._ck(self.L.oracle_artifact_info(data, len(data), ctypes.byref(m), ctypes.byref(n), ctypes.byref(s)))
        return m.value, n.value, s.value

    def infer(self, data: bytes, x: np.ndarray, threads: int = 1) -> np.ndarray:
        m, n, _ = self.artifact_info(data)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, n)
        y = np.zeros((x.shape[0], m))
        self._ck(self.L.oracle_infer(data, len(data), _ptr(x), x.shape[0], _ptr(y), threads))
        return y

    def decode_stage(self, data: bytes, stage: int) -> np.ndarray:
        m, n, _ = self.artifact_info(data)
        w = np.zeros((m, n))
        self._ck(self.L.oracle_decode_stage(data, len(data), stage, _ptr(w)))
        return w


def build_oracle(ref: bool = False) -> None:
    """make -C oracle oracle [ref] (ref needs /root/reference)."""
    import subprocess
    targets = ["oracle"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)
