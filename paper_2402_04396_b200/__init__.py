"""q8p: B200-native (sm_100a) QuIP# quantized-linear inference.

Python mirror of the reference `latq` inference-path interface
(/root/reference/proj/core/include/latq/pipeline.hpp: QuantizedLinear,
infer, serialize/deserialize; hadamard.hpp: plan_hadamard), bound over the
C ABI in include/q8p.h (libq8p.so, built in-tree by __graft_entry__.build()).

There is no CPU fallback: every compute call runs the sm_100a kernels and
fails loudly when the extension or a B200 is missing.  torch is used only
for device memory and streams.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "LayerSet", "Error", "SizeError", "ValidationError", "FormatError", "BadMagicError",
    "UnsupportedVersionError", "TruncatedArtifactError", "UnsupportedError", "DeviceError",
    "lib", "plan_hadamard", "hadamard_base", "codebook_table", "e8p_decode_host",
    "inspect_artifact", "reserialize", "Layer", "rht", "kernel_launches", "e8p_encode", "rvq_quantize", "rht_cols_f64",
    "CB_E8P_2BIT", "CB_E8_1BIT", "NcclError", "shard_rows", "NcclComm",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# Q8P_LIB: an alternative in-tree build of the same library (experiment builds)
LIB_PATH = os.environ.get("Q8P_LIB") or os.path.join(_HERE, "libq8p.so")

CB_E8P_2BIT = 0
CB_E8_1BIT = 1


# --- error taxonomy (core/include/latq/errors.hpp:9-53) ---------------------
class Error(RuntimeError):
    pass


class SizeError(Error):
    pass


class ValidationError(Error):
    pass


class FormatError(Error):
    pass


class BadMagicError(FormatError):
    pass


class UnsupportedVersionError(FormatError):
    pass


class TruncatedArtifactError(FormatError):
    pass


class UnsupportedError(Error):
    pass


class DeviceError(Error):
    pass


class NcclError(DeviceError):
    pass


_STATUS = {
    1: SizeError, 2: ValidationError, 3: FormatError, 4: BadMagicError,
    5: UnsupportedVersionError, 6: TruncatedArtifactError, 7: UnsupportedError,
    8: DeviceError, 9: NcclError, 10: Error,
}


class LayerDesc(ctypes.Structure):
    pass


class StageDesc(ctypes.Structure):
    _fields_ = [("codebook", ctypes.c_int), ("scale", ctypes.c_float),
                ("codes", ctypes.c_void_p), ("code_bytes", ctypes.c_int)]


LayerDesc._fields_ = [("m", ctypes.c_uint32), ("n", ctypes.c_uint32), ("transform", ctypes.c_int),
                      ("num_stages", ctypes.c_int), ("stages", ctypes.POINTER(StageDesc)),
                      ("signs_u", ctypes.c_void_p), ("signs_v", ctypes.c_void_p),
                      ("phases_u", ctypes.c_void_p), ("phases_v", ctypes.c_void_p)]


class ForwardOpts(ctypes.Structure):
    _fields_ = [("gemv_start_event", ctypes.c_void_p), ("gemv_end_event", ctypes.c_void_p)]


class LayerInfo(ctypes.Structure):
    _fields_ = [("m", ctypes.c_uint32), ("n", ctypes.c_uint32), ("row_begin", ctypes.c_uint32),
                ("row_end", ctypes.c_uint32), ("num_stages", ctypes.c_int), ("device", ctypes.c_int),
                ("device_bytes", ctypes.c_size_t), ("code_bytes", ctypes.c_size_t)]


class ArtifactInfo(ctypes.Structure):
    _fields_ = [("m", ctypes.c_uint32), ("n", ctypes.c_uint32), ("transform", ctypes.c_int),
                ("num_stages", ctypes.c_int), ("codebook", ctypes.c_int * 8),
                ("scale", ctypes.c_float * 8), ("serialized_size", ctypes.c_size_t)]


# Every symbol include/q8p.h declares, with its ctypes signature.
_SIGNATURES = {
    "q8p_version": (ctypes.c_char_p, []),
    "q8p_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "q8p_last_error": (ctypes.c_char_p, []),
    "q8p_kernel_launches": (ctypes.c_uint64, []),
    "q8p_plan_hadamard": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]),
    "q8p_layer_create": (ctypes.c_int, [ctypes.POINTER(LayerDesc), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "q8p_layer_from_qshp": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "q8p_layer_from_qshp_rows": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "q8p_layer_destroy": (None, [ctypes.c_void_p]),
    "q8p_layer_get_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(LayerInfo)]),
    "q8p_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int]),
    "q8p_forward": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "q8p_forward_ex": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.POINTER(ForwardOpts)]),
    "q8p_forward_rows_z": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "q8p_forward_sharded": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]),
    "q8p_infer_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "q8p_e8p_encode": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]),
    "q8p_rvq_quantize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "q8p_rht_cols_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                        ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "q8p_forward_set_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    "q8p_forward_set_workspace_bytes_ex": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint]),
    "q8p_forward_set_ex": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_uint]),
    "q8p_forward_set_host_ex": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                               ctypes.c_uint]),
    "q8p_forward_set": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "q8p_forward_set_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                            ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "q8p_decode_stage": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "q8p_bench_gemv": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]),
    "q8p_bench_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]),
    "q8p_layer_code_region": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]),
    "q8p_forward_sharded_sim": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "q8p_dequantize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "q8p_k2_decode_stage": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "q8p_rht": (ctypes.c_int, [ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    "q8p_qshp_inspect": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ArtifactInfo)]),
    "q8p_qshp_reserialize": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "q8p_e8p_decode_host": (ctypes.c_int, [ctypes.c_uint16, ctypes.c_void_p]),
    "q8p_codebook_table": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "q8p_hadamard_base": (ctypes.c_int, [ctypes.c_size_t, ctypes.c_void_p]),
    "q8p_layers_from_qshp": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    "q8p_peers_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]),
    "q8p_peers_connect": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p]),
    "q8p_peers_connect_local": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "q8p_peers_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "q8p_peers_state": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "q8p_forward_sharded_push": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "q8p_forward_sharded_push_sim": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "q8p_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "q8p_nccl_comm_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "q8p_nccl_comm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
}

_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Load libq8p.so (built in-tree).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"q8p extension not built: {LIB_PATH} missing "
                              "(run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            if os.environ.get("Q8P_LIB") and not hasattr(L, name):
                continue  # an older experiment build: entry points it lacks stay unbound
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        msg = lib().q8p_last_error().decode(errors="replace")
        raise _STATUS.get(status, Error)(msg)


def kernel_launches() -> int:
    return int(lib().q8p_kernel_launches())


# --- host-side helpers (no GPU) ----------------------------------------------
def plan_hadamard(n: int) -> tuple[int, int]:
    """latq::plan_hadamard (hadamard.cpp:156-168), registry + 172 -> (p, q)."""
    p, q = ctypes.c_size_t(), ctypes.c_size_t()
    _check(lib().q8p_plan_hadamard(n, ctypes.byref(p), ctypes.byref(q)))
    return p.value, q.value


def hadamard_base(q: int) -> np.ndarray:
    out = np.zeros(q * q, dtype=np.int8)
    _check(lib().q8p_hadamard_base(q, out.ctypes.data))
    return out.reshape(q, q)


def codebook_table(cb: int) -> tuple[np.ndarray, np.ndarray]:
    d = np.zeros((256, 8), dtype=np.int8)
    p = np.zeros(256, dtype=np.uint8)
    _check(lib().q8p_codebook_table(cb, d.ctypes.data, p.ctypes.data))
    return d, p


def e8p_decode_host(word: int) -> np.ndarray:
    out = np.zeros(8, dtype=np.float32)
    _check(lib().q8p_e8p_decode_host(word, out.ctypes.data))
    return out


def inspect_artifact(data: bytes) -> dict:
    info = ArtifactInfo()
    _check(lib().q8p_qshp_inspect(data, len(data), ctypes.byref(info)))
    return {"m": info.m, "n": info.n, "transform": info.transform, "num_stages": info.num_stages,
            "codebook": list(info.codebook[: info.num_stages]), "scale": list(info.scale[: info.num_stages]),
            "serialized_size": info.serialized_size}


def reserialize(data: bytes) -> bytes:
    """serialize(deserialize(data)) through the product's QSHP reader/writer."""
    n = ctypes.c_size_t()
    buf = ctypes.create_string_buffer(len(data) + 64)
    _check(lib().q8p_qshp_reserialize(data, len(data), buf, len(buf), ctypes.byref(n)))
    return buf.raw[: n.value]


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Row shard [lo, hi) of rank `rank` for q8p_forward_sharded: equal shards,
    ordered by rank (the all-gather's rank-major layout is then z itself)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValidationError(f"bad world/rank {world}/{rank}")
    if m % world:
        raise ValidationError(f"m={m} is not divisible by world={world}")
    per = m // world
    return rank * per, (rank + 1) * per


class NcclComm:
    """NCCL communicator for Layer.forward_sharded (q8p_nccl_* plumbing: the
    unique id is broadcast by the caller, e.g. over torch.distributed)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().q8p_nccl_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, world: int, rank: int, device: int):
        if len(uid) != 128:
            raise ValidationError("NCCL unique id must be 128 bytes")
        c = ctypes.c_void_p()
        _check(lib().q8p_nccl_comm_init(uid, world, rank, device, ctypes.byref(c)))
        self.handle = c
        self.world, self.rank = world, rank

    def close(self) -> None:
        if self.handle:
            _check(lib().q8p_nccl_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


PEER_HANDLE_BYTES = 64


class PeerGroup:
    """One rank's member of a push all-gather group (q8p_peers_*): a window in
    this GPU's memory that the other ranks write into over NVLink.  Exchange
    `handle` (bytes) among the ranks out of band, then `connect(handles)` with the
    rank-ordered list.  slice_floats >= min(batch, 32) * m_local of every layer used
    (batch * m_local for prefill batches >= 64)."""

    def __init__(self, device: int, world: int, rank: int, slice_floats: int):
        h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * PEER_HANDLE_BYTES)()
        _check(lib().q8p_peers_create(device, world, rank, slice_floats, ctypes.byref(h), buf))
        self._h = h
        self.handle = bytes(buf)
        self.device, self.world, self.rank = device, world, rank

    def connect(self, handles) -> None:
        if len(handles) != self.world or any(len(b) != PEER_HANDLE_BYTES for b in handles):
            raise ValidationError(f"need {self.world} handles of {PEER_HANDLE_BYTES} bytes")
        _check(lib().q8p_peers_connect(self._h, b"".join(handles)))

    @staticmethod
    def connect_local(group) -> None:
        """Wire the members of one group created in this process (tests, one GPU)."""
        arr = (ctypes.c_void_p * len(group))(*[g._h.value for g in group])
        _check(lib().q8p_peers_connect_local(arr, len(group)))

    def state(self) -> int:
        """Push calls (K3 chunks) completed on this rank."""
        ep = ctypes.c_uint64()
        _check(lib().q8p_peers_state(self._h, ctypes.byref(ep)))
        return ep.value

    def close(self) -> None:
        if self._h:
            _check(lib().q8p_peers_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --- device API ---------------------------------------------------------------
def _torch():
    import torch  # plumbing only: device memory and streams
    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Layer:
    """A QuantizedLinear resident on one B200 (or a row shard of one)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)
        self._ws = None

    @classmethod
    def from_qshp(cls, data: bytes, device: int = 0, rows: Optional[tuple[int, int]] = None) -> "Layer":
        h = ctypes.c_void_p()
        if rows is None:
            _check(lib().q8p_layer_from_qshp(data, len(data), device, ctypes.byref(h)))
        else:
            _check(lib().q8p_layer_from_qshp_rows(data, len(data), rows[0], rows[1], device, ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def many_from_qshp(cls, artifacts: Sequence[bytes], device: int = 0) -> list["Layer"]:
        """q8p_layers_from_qshp: a model's artifacts loaded concurrently (parse / H2D /
        device transcode of different layers overlap)."""
        k = len(artifacts)
        arts = [bytes(a) for a in artifacts]  # no copy for bytes; kept alive for the call
        ptrs = (ctypes.c_char_p * k)(*arts)
        lens = (ctypes.c_size_t * k)(*[len(a) for a in artifacts])
        out = (ctypes.c_void_p * k)()
        _check(lib().q8p_layers_from_qshp(ptrs, lens, k, device, out))
        return [cls(out[i]) for i in range(k)]

    @classmethod
    def create(cls, m: int, n: int, stages: Sequence[tuple[int, float, np.ndarray]],
               signs_u: np.ndarray | None = None, signs_v: np.ndarray | None = None, device: int = 0,
               phases_u: np.ndarray | None = None, phases_v: np.ndarray | None = None) -> "Layer":
        """q8p_layer_create from raw fields: stages = [(codebook, scale, codes)];
        sign bytes (rht) or f32 phase angles (rfft, m/2 and n/2 of them)."""
        st = (StageDesc * len(stages))()
        keep = []
        for i, (cb, scale, codes) in enumerate(stages):
            codes = np.ascontiguousarray(codes)
            keep.append(codes)
            st[i].codebook = cb
            st[i].scale = scale
            st[i].codes = codes.ctypes.data
            st[i].code_bytes = codes.dtype.itemsize
        rfft = phases_u is not None or phases_v is not None
        if rfft:
            pu = np.ascontiguousarray(phases_u, dtype=np.float32)
            pv = np.ascontiguousarray(phases_v, dtype=np.float32)
            keep += [pu, pv]
            d = LayerDesc(m, n, 1, len(stages), st, None, None, pu.ctypes.data, pv.ctypes.data)
        else:
            su = np.ascontiguousarray(signs_u, dtype=np.uint8)
            sv = np.ascontiguousarray(signs_v, dtype=np.uint8)
            keep += [su, sv]
            d = LayerDesc(m, n, 0, len(stages), st, su.ctypes.data, sv.ctypes.data, None, None)
        h = ctypes.c_void_p()
        _check(lib().q8p_layer_create(ctypes.byref(d), device, ctypes.byref(h)))
        return cls(h.value)

    def close(self) -> None:
        if self._h and self._h.value:
            lib().q8p_layer_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def info(self) -> dict:
        i = LayerInfo()
        _check(lib().q8p_layer_get_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in LayerInfo._fields_}

    def workspace_bytes(self, batch: int) -> int:
        return int(lib().q8p_workspace_bytes(self._h, batch))

    def workspace(self, batch: int):
        torch = _torch()
        need = self.workspace_bytes(batch)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.info['device']}")
        return self._ws

    def _dims(self):
        d = self.__dict__.get("_dims_cache")
        if d is None:  # immutable after creation: query the C ABI once
            i = self.info
            d = self.__dict__["_dims_cache"] = (i["m"], i["n"])
        return d

    def _check_x(self, x, n):
        torch = _torch()
        if x.dim() != 2 or x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
            raise ValidationError("x must be a contiguous float32 CUDA tensor [batch, n]")
        if x.device.index != self.info["device"]:
            raise ValidationError("x is on another device than the layer")
        if x.shape[1] != n:
            raise SizeError("infer: input length != n")

    @staticmethod
    def _out(out, x, rows):
        torch = _torch()
        if out is None:
            return torch.empty(x.shape[0], rows, dtype=torch.float32, device=x.device)
        if (out.dtype != torch.float32 or not out.is_contiguous() or out.device != x.device
                or tuple(out.shape) != (x.shape[0], rows)):
            raise ValidationError(f"out must be a contiguous float32 tensor [{x.shape[0]}, {rows}] on x's device")
        return out

    def forward(self, x, out=None, stream=None, workspace=None, gemv_events=None):
        """y = W_tilde x for a [batch, n] fp32 CUDA tensor -> [batch, m].
        gemv_events: optional (start, end) torch.cuda.Event pair recorded
        around the decode-GEMV kernel."""
        m, n = self._dims()
        if x.dim() == 1:
            return self.forward(x.view(1, -1), None if out is None else out.view(1, -1), stream, workspace,
                                gemv_events).view(-1)
        self._check_x(x, n)
        batch = x.shape[0]
        out = self._out(out, x, m)
        ws = workspace if workspace is not None else self.workspace(batch)
        if gemv_events is None:
            _check(lib().q8p_forward(self._h, x.data_ptr(), out.data_ptr(), batch, ws.data_ptr(),
                                     ws.numel(), _stream_ptr(stream)))
        else:
            opts = ForwardOpts(gemv_events[0].cuda_event, gemv_events[1].cuda_event)
            _check(lib().q8p_forward_ex(self._h, x.data_ptr(), out.data_ptr(), batch, ws.data_ptr(),
                                        ws.numel(), _stream_ptr(stream), ctypes.byref(opts)))
        return out

    def rows_z(self, x, stream=None, workspace=None):
        """This handle's rows of z = W_hat T_v x ([batch, rows]); the slice a
        row-sharded forward all-gathers before y = T_u^T z."""
        info = self.info
        self._check_x(x, info["n"])
        batch = x.shape[0]
        z = self._out(None, x, info["row_end"] - info["row_begin"])
        ws = workspace if workspace is not None else self.workspace(batch)
        _check(lib().q8p_forward_rows_z(self._h, x.data_ptr(), z.data_ptr(), batch, ws.data_ptr(), ws.numel(),
                                        _stream_ptr(stream)))
        return z

    def forward_sharded(self, x, comm, out=None, stream=None, workspace=None):
        """Row-sharded forward (q8p_forward_sharded): this layer holds rows
        shard_rows(m, world, rank); z slices are all-gathered over `comm`
        (NcclComm or a raw ncclComm_t pointer) and every rank gets the full y."""
        if isinstance(comm, NcclComm):
            comm = comm.handle
        info = self.info
        self._check_x(x, info["n"])
        batch = x.shape[0]
        out = self._out(out, x, info["m"])
        ws = workspace if workspace is not None else self.workspace(batch)
        _check(lib().q8p_forward_sharded(self._h, x.data_ptr(), out.data_ptr(), batch, ws.data_ptr(),
                                         ws.numel(), comm, _stream_ptr(stream)))
        return out

    def forward_sharded_push(self, x, peers: "PeerGroup", out=None, stream=None, workspace=None):
        """Row-sharded forward with the all-gather fused into K3 pass 1
        (q8p_forward_sharded_push): every rank's rows are pushed into every rank's
        PeerGroup window over NVLink; every rank gets the full y."""
        info = self.info
        self._check_x(x, info["n"])
        batch = x.shape[0]
        out = self._out(out, x, info["m"])
        ws = workspace if workspace is not None else self.workspace(batch)
        _check(lib().q8p_forward_sharded_push(self._h, peers._h, x.data_ptr(), out.data_ptr(), batch, ws.data_ptr(),
                                              ws.numel(), _stream_ptr(stream)))
        return out

    def infer_host(self, x: np.ndarray) -> np.ndarray:
        """latq::infer calling convention: host f64 [batch, n] -> host f64 [batch, m]."""
        info = self.info
        x = np.ascontiguousarray(x, dtype=np.float64)
        squeeze = x.ndim == 1
        x2 = x.reshape(-1, info["n"]) if x.size % max(info["n"], 1) == 0 else None
        if x2 is None or (squeeze and x.shape[0] != info["n"]):
            raise SizeError("infer: input length != n")
        y = np.zeros((x2.shape[0], info["m"]), dtype=np.float64)
        _check(lib().q8p_infer_host(self._h, x2.ctypes.data, y.ctypes.data, x2.shape[0]))
        return y[0] if squeeze else y

    def bench_gemv(self, batch: int, workspace, reps: int, stream=None):
        """`reps` back-to-back K2 launches on the B images in `workspace` (q8p_bench_gemv)."""
        _check(lib().q8p_bench_gemv(self._h, batch, workspace.data_ptr(), workspace.numel(), reps, _stream_ptr(stream)))

    def code_region(self, stage: int = 0):
        """(device address, bytes) of a stage's code slabs (q8p_layer_code_region)."""
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().q8p_layer_code_region(self._h, stage, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def dequantize(self, stream=None):
        """latq::dequantize_layer on the device (q8p_dequantize): dense W~ [m, n] float64."""
        torch = _torch()
        info = self.info
        dev = f"cuda:{info['device']}"
        w = torch.empty(info["m"], info["n"], dtype=torch.float64, device=dev)
        scratch = torch.empty_like(w)
        _check(lib().q8p_dequantize(self._h, w.data_ptr(), scratch.data_ptr(), _stream_ptr(stream)))
        return w

    def k2_decode_stage(self, stage: int, stream=None):
        """The GEMV kernel's own operand decode of one stage (q8p_k2_decode_stage):
        (a int8 [m_local][n], shift uint8 [m_local][n/8] or None for e8-1bit)."""
        torch = _torch()
        info = self.info
        ml = info["row_end"] - info["row_begin"]
        a = torch.empty(ml, info["n"], dtype=torch.int8, device=f"cuda:{info['device']}")
        sh = torch.zeros(ml, info["n"] // 8, dtype=torch.uint8, device=a.device)
        _check(lib().q8p_k2_decode_stage(self._h, stage, a.data_ptr(), sh.data_ptr(), _stream_ptr(stream)))
        return a, sh

    def decode_stage(self, stage: int, stream=None):
        torch = _torch()
        info = self.info
        w = torch.empty(info["row_end"] - info["row_begin"], info["n"], dtype=torch.float32,
                        device=f"cuda:{info['device']}")
        _check(lib().q8p_decode_stage(self._h, stage, w.data_ptr(), _stream_ptr(stream)))
        return w


SET_CONCURRENT = 1  # Q8P_SET_CONCURRENT


class LayerSet:
    """Independent layer forwards per call (q8p_forward_set_ex / _host_ex): one
    decode step through a model's linear layers.  concurrent=True: the layers
    read only their own inputs and run on parallel streams (Q8P_SET_CONCURRENT)."""

    def __init__(self, layers: Sequence[Layer], concurrent: bool = False):
        self.flags = SET_CONCURRENT if concurrent else 0
        self.layers = list(layers)  # keeps the handles alive
        self._arr = (ctypes.c_void_p * len(self.layers))(*[L._h.value for L in self.layers])
        self._ws = None
        self._nsum = sum(L._dims()[1] for L in self.layers)
        self._msum = sum(L._dims()[0] for L in self.layers)

    def workspace_bytes(self, batch: int) -> int:
        return int(lib().q8p_forward_set_workspace_bytes_ex(self._arr, len(self.layers), batch, self.flags))

    def workspace(self, batch: int):
        torch = _torch()
        need = self.workspace_bytes(batch)
        if self._ws is None or self._ws.numel() < need:
            dev = self.layers[0].info["device"]
            self._ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{dev}")
        return self._ws

    def forward(self, xs, outs=None, stream=None, workspace=None):
        """xs: [batch, n_i] fp32 CUDA tensors -> [batch, m_i] tensors."""
        torch = _torch()
        batch = xs[0].shape[0]
        if outs is None:
            outs = [torch.empty(batch, L._dims()[0], dtype=torch.float32, device=x.device)
                    for L, x in zip(self.layers, xs)]
        for L, x, y in zip(self.layers, xs, outs):
            if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous() or x.shape != (batch, L._dims()[1]):
                raise ValidationError("xs[i] must be contiguous float32 CUDA [batch, n_i]")
            if y.shape != (batch, L._dims()[0]) or not y.is_contiguous():
                raise ValidationError("outs[i] must be contiguous [batch, m_i]")
        xp = (ctypes.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
        yp = (ctypes.c_void_p * len(outs))(*[y.data_ptr() for y in outs])
        ws = workspace if workspace is not None else self.workspace(batch)
        _check(lib().q8p_forward_set_ex(self._arr, len(self.layers), xp, yp, batch, ws.data_ptr(), ws.numel(),
                                        _stream_ptr(stream), self.flags))
        return outs

    def forward_host(self, x_host, y_host, batch: int, stream=None, workspace=None):
        """Host fp32 buffers (torch CPU tensors, pinned for the graph path):
        x_host = inputs concatenated [i][batch][n_i], y_host = outputs [i][batch][m_i].
        Returns when y_host holds the results."""
        if x_host.numel() < batch * self._nsum or y_host.numel() < batch * self._msum:
            raise SizeError("host buffers too small for the layer set")
        ws = workspace if workspace is not None else self.workspace(batch)
        st = lib().q8p_forward_set_host_ex(self._arr, len(self._arr), x_host.data_ptr(), y_host.data_ptr(), batch,
                                           ws.data_ptr(), ws.numel(), _stream_ptr(stream), self.flags)
        if st:
            _check(st)
        return y_host


def e8p_encode(v, stream=None):
    """Nearest E8P codewords of a float64 CUDA tensor [nblocks, 8] (reference
    e8p_encode, bit-identical) -> int32 tensor [nblocks] of 16-bit words."""
    torch = _torch()
    if v.dtype != torch.float64 or not v.is_cuda or not v.is_contiguous() or v.dim() != 2 or v.shape[1] != 8:
        raise ValidationError("v must be a contiguous float64 CUDA tensor [nblocks, 8]")
    out = torch.empty(v.shape[0], dtype=torch.int16, device=v.device)
    _check(lib().q8p_e8p_encode(v.data_ptr(), out.data_ptr(), v.shape[0], v.device.index or 0, _stream_ptr(stream)))
    return out.to(torch.int32) & 0xFFFF


def rvq_quantize(v, stages, stream=None):
    """RvqQuantizer::quantize on a float64 CUDA tensor [nblocks, 8]; stages =
    [(codebook, scale)] (CB_E8P_2BIT / CB_E8_1BIT, float scale) -> int32 codes
    [num_stages, nblocks] (bit-identical to the reference)."""
    torch = _torch()
    if v.dtype != torch.float64 or not v.is_cuda or not v.is_contiguous() or v.dim() != 2 or v.shape[1] != 8:
        raise ValidationError("v must be a contiguous float64 CUDA tensor [nblocks, 8]")
    out = torch.empty(len(stages), v.shape[0], dtype=torch.int16, device=v.device)
    cbs = (ctypes.c_int * len(stages))(*[int(cb) for cb, _ in stages])
    scs = (ctypes.c_double * len(stages))(*[float(sc) for _, sc in stages])
    _check(lib().q8p_rvq_quantize(v.data_ptr(), out.data_ptr(), v.shape[0], len(stages), cbs, scs,
                                  v.device.index or 0, _stream_ptr(stream)))
    return out.to(torch.int32) & 0xFFFF


def forward_sharded_sim(shards, x, stream=None):
    """q8p_forward_sharded_sim: the row-sharded forward of `shards` (rank-ordered
    row-range handles of one layer on one GPU) with the all-gather simulated by copies."""
    torch = _torch()
    info = shards[0].info
    shards[0]._check_x(x, info["n"])
    y = torch.empty(x.shape[0], info["m"], dtype=torch.float32, device=x.device)
    ws = shards[0].workspace(x.shape[0])
    arr = (ctypes.c_void_p * len(shards))(*[S._h.value for S in shards])
    _check(lib().q8p_forward_sharded_sim(arr, len(shards), x.data_ptr(), y.data_ptr(), x.shape[0], ws.data_ptr(),
                                         ws.numel(), _stream_ptr(stream)))
    return y


def forward_sharded_push_sim(shards, peers, x, stream=None):
    """q8p_forward_sharded_push_sim: every rank's push forward on one GPU (peers
    wired by PeerGroup.connect_local); returns [world, batch, m] (each rank's y)."""
    torch = _torch()
    info = shards[0].info
    shards[0]._check_x(x, info["n"])
    y = torch.empty(len(shards), x.shape[0], info["m"], dtype=torch.float32, device=x.device)
    ws = shards[0].workspace(x.shape[0])
    arr = (ctypes.c_void_p * len(shards))(*[S._h.value for S in shards])
    parr = (ctypes.c_void_p * len(peers))(*[p._h.value for p in peers])
    _check(lib().q8p_forward_sharded_push_sim(arr, parr, len(shards), x.data_ptr(), y.data_ptr(), x.shape[0],
                                              ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
    return y


def bench_stream(addr: int, nbytes: int, reps: int, stream=None):
    """`reps` plain HBM reads of [addr, addr + nbytes) in K2's access pattern (q8p_bench_stream)."""
    _check(lib().q8p_bench_stream(ctypes.c_void_p(addr), nbytes, reps, _stream_ptr(stream)))


def rht_cols_f64(w, signs, stream=None):
    """SideTransform::apply (rht) on every column of a contiguous float64 CUDA
    matrix [rows, cols], in place; signs: uint8 CUDA tensor of ceil(rows/8)
    bytes.  Bit-identical to the reference's transform_cols."""
    torch = _torch()
    if w.dtype != torch.float64 or not w.is_cuda or not w.is_contiguous() or w.dim() != 2:
        raise ValidationError("w must be a contiguous float64 CUDA matrix")
    scratch = torch.empty_like(w)
    _check(lib().q8p_rht_cols_f64(w.data_ptr(), scratch.data_ptr(), w.shape[0], w.shape[1], signs.data_ptr(),
                                  w.device.index or 0, _stream_ptr(stream)))
    return w


def rht(x, signs, transpose: bool = False, out=None, stream=None):
    """SideTransform apply / apply_transpose on [batch, n] fp32 CUDA tensors;
    signs: uint8 CUDA tensor of ceil(n/8) bytes."""
    torch = _torch()
    if x.dim() == 1:
        x = x.view(1, -1)
    if out is None:
        out = torch.empty_like(x)
    _check(lib().q8p_rht(x.shape[1], signs.data_ptr(), x.data_ptr(), out.data_ptr(), x.shape[0],
                         1 if transpose else 0, _stream_ptr(stream)))
    return out


# RVQ schemes of the reference producer (rvq.cpp:9-21): codebook ids and rho_i.
RVQ_SCHEMES = {2: (["e8p-2bit"], [0.9]), 3: (["e8p-2bit", "e8-1bit"], [0.98, 2.04]),
               4: (["e8p-2bit", "e8p-2bit"], [1.03, 3.45])}


def produce_artifact(w, signs_u, signs_v, bits: int, exact_r1: bool = True) -> bytes:
    """GPU producer: the reference's H = I quantize_layer route
    (pipeline.cpp:47-107 with ldlq.cpp's nearest rounding) on a float64 CUDA weight
    matrix w [m, n] and host sign-byte arrays -> QSHP v1 bytes, byte-identical to the
    reference artifact for the same W and signs (tests/test_gpu_encode.py):
    W~ = T_u W T_v^T in f64 (q8p_rht_cols_f64), r1 = ||W~|| / sqrt(mn) (column-major,
    left-to-right sum as the reference), f32-frozen stage scales r1 / rho_i, RVQ codes
    (q8p_rvq_quantize).  w is consumed (transformed in place).  exact_r1=False sums
    ||W~||^2 on the device instead (last-ulp differences in r1; for synthetic
    benchmark weights only)."""
    import struct

    import numpy as np
    torch = _torch()
    m, n = w.shape
    if bits not in RVQ_SCHEMES:
        raise ValidationError("bits must be 2, 3 or 4")
    su = torch.from_numpy(np.ascontiguousarray(signs_u, dtype=np.uint8)).to(w.device)
    sv = torch.from_numpy(np.ascontiguousarray(signs_v, dtype=np.uint8)).to(w.device)
    rht_cols_f64(w, su)                          # transform_cols(left)
    wt = w.t().contiguous()
    rht_cols_f64(wt, sv)                         # transform_rows(right)
    wt = wt.t().contiguous()
    if exact_r1:
        sq = (wt.t().contiguous().view(-1) ** 2).cpu().numpy()
        r1 = np.sqrt(np.cumsum(sq)[-1]) / np.sqrt(float(m) * n)
    else:
        r1 = float(torch.sqrt((wt * wt).sum())) / np.sqrt(float(m) * n)
    ids, rho = RVQ_SCHEMES[bits]
    s32 = [np.float32(r1 / r) for r in rho]
    cbs = [CB_E8P_2BIT if i == "e8p-2bit" else CB_E8_1BIT for i in ids]
    codes = rvq_quantize(wt.view(-1, 8), list(zip(cbs, [float(x) for x in s32]))).cpu().numpy()
    body = b"QSHP" + struct.pack("<HIIBB", 1, m, n, 0, len(ids))
    for i, sc in zip(ids, s32):
        body += bytes([len(i)]) + i.encode() + struct.pack("<f", sc)
    body += np.ascontiguousarray(signs_u, dtype=np.uint8).tobytes() + np.ascontiguousarray(signs_v, dtype=np.uint8).tobytes()
    for cid, c in zip(ids, codes):
        body += c.astype("<u2" if cid == "e8p-2bit" else "u1").tobytes()
    return body
