"""B200-native HCInfer compensated quantized linear (arXiv 2605.05819).

Thin Python binding over the C-ABI library ``libhcinfer.so`` (include/hcinfer.h).  Names
follow the C entry points: ``allocate_ranks``, ``Context.load_layer``, ``Context.set_rank``,
``Context.compensated_linear``.  This module only marshals arguments (numpy arrays or torch
tensors -> raw pointers, the current torch CUDA stream -> cudaStream_t); PyTorch is used for
device memory and streams only.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (HCError, HC_OK, HC_ERR_CONFIG, HC_ERR_STATE, HC_ERR_NUMERIC, HC_ERR_RUNTIME,
                   QKV, O, UPGATE, DOWN, OUT_F32, OUT_BF16, GLUE_NONE, GLUE_SILU_MUL, FACTORS_BF16, FACTORS_FP8,
                   check, lib)

__all__ = ["allocate_ranks", "Context", "HCError", "QKV", "O", "UPGATE", "DOWN", "OUT_F32", "OUT_BF16",
           "GLUE_NONE", "GLUE_SILU_MUL", "FACTORS_BF16", "FACTORS_FP8",
           "repack_host", "unpack_repacked_host", "shard_rows", "unshard_host", "set_option", "get_option", "calib_r_std", "lib"]


def calib_r_std(Ns, K, bits, group=128, eps=0.1) -> float:
    """hc_calib_r_std: B200 byte-budget r_std of a window (R17)."""
    arr = np.ascontiguousarray(Ns, dtype=np.int32)
    out = C.c_double(0.0)
    check(lib().hc_calib_r_std(arr.ctypes.data, int(arr.size), int(K), int(bits), int(group), float(eps), C.addressof(out)))
    return float(out.value)


def set_option(name: str, value: int) -> None:
    """hc_set_option: process-wide development switch (include/hcinfer.h lists them)."""
    check(lib().hc_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    """hc_get_option."""
    v = C.c_int32(0)
    check(lib().hc_get_option(name.encode(), C.addressof(v)))
    return int(v.value)


def shard_rows(N: int, world: int, rank: int, unit: int = 16):
    """Column sharding of a weight matrix's output rows: rank p keeps rows
    [p·N/G, (p+1)·N/G).  N/G must be a multiple of `unit` (16 = the kernel's row block)."""
    if N % world or (N // world) % unit:
        raise ValueError(f"N={N} cannot be column-sharded over {world} ranks in {unit}-row units")
    n = N // world
    return rank * n, (rank + 1) * n


def _ptr(a):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous(), "tensors must be contiguous"
        return a.data_ptr()
    raise TypeError(type(a))


def _itemsize(a) -> int:
    return a.itemsize if isinstance(a, np.ndarray) else a.element_size()


def _check_buf(name, a, n_elems, sizes, what):
    """Argument check before a raw pointer crosses the ABI: element size in `sizes` and at least n_elems
    elements (the C side trusts both)."""
    if _itemsize(a) not in sizes:
        raise TypeError(f"{name}: expected {what} (element size {sizes}), got element size {_itemsize(a)}")
    n = a.size if isinstance(a, np.ndarray) else a.numel()
    if n < n_elems:
        raise ValueError(f"{name}: {n} elements < the {n_elems} the call reads / writes")


def _is_int32(a) -> bool:
    return (a.dtype == np.int32) if isinstance(a, np.ndarray) else str(a.dtype) == "torch.int32"


def _is_f32(a) -> bool:
    return (a.dtype == np.float32) if isinstance(a, np.ndarray) else str(a.dtype) == "torch.float32"


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


# ------------------------------------------------------------------ allocation (host)
def allocate_ranks(records, D_layer, top_k_layers, r_std, caps, tau=0.01, k0=3, two_stage_mode=0, moe_k=0):
    """hc_allocate_ranks.  records: iterable of dicts with keys layer, window, slot, expert,
    sigma (array or None), phi, n_sal, n_all, D, gate.  Returns (ranks int32, priority float64)."""
    recs = list(records)
    n = len(recs)
    arr = (_lib.hc_sens * max(n, 1))()
    keep = []
    for i, r in enumerate(recs):
        s = arr[i]
        s.layer, s.window_kind, s.slot = int(r["layer"]), int(r["window"]), int(r["slot"])
        s.expert = int(r.get("expert", -1))
        sig = r.get("sigma")
        if sig is not None:
            sig = np.ascontiguousarray(sig, dtype=np.float64)
            keep.append(sig)
            s.n_sigma, s.sigma = sig.size, sig.ctypes.data_as(C.POINTER(C.c_double))
        else:
            s.n_sigma, s.sigma = 0, None
        s.phi = float(r.get("phi", 1.0))
        s.n_salient, s.n_total = int(r.get("n_sal", 0)), int(r.get("n_all", 0))
        s.D_matrix, s.gate = float(r["D"]), float(r.get("gate", 1.0))
    dl = np.ascontiguousarray(D_layer, dtype=np.float64)
    b = _lib.hc_budget()
    b.n_layers, b.D_layer = dl.size, dl.ctypes.data_as(C.POINTER(C.c_double))
    b.top_k_layers, b.tau, b.k0 = int(top_k_layers), float(tau), int(k0)
    for k in range(4):
        b.r_std[k] = float(r_std[k])
    b.two_stage_mode, b.moe_k = int(two_stage_mode), int(moe_k)
    capv = np.ascontiguousarray(caps, dtype=np.int32)
    ranks = np.zeros(max(n, 1), dtype=np.int32)
    prio = np.zeros(max(n, 1), dtype=np.float64)
    check(lib().hc_allocate_ranks(arr, n, C.byref(b), capv.ctypes.data_as(C.POINTER(C.c_int32)),
                                  ranks.ctypes.data_as(C.POINTER(C.c_int32)),
                                  prio.ctypes.data_as(C.POINTER(C.c_double))))
    return ranks[:n], prio[:n]


# ------------------------------------------------------------------ layout test exports (host)
def repack_host(codes, scales, zeros, N, K, bits):
    out = np.zeros(lib().hc_repacked_bytes(N, K, bits), dtype=np.uint8)
    check(lib().hc_repack_host(_ptr(codes), _ptr(scales), _ptr(zeros), N, K, bits, _ptr(out)))
    return out


def unpack_repacked_host(packed, N, K, bits):
    q = np.zeros((N, K), dtype=np.uint8)
    s = np.zeros((N, K // 128), dtype=np.uint16)
    z = np.zeros((N, K // 128), dtype=np.uint8)
    check(lib().hc_unpack_repacked_host(_ptr(packed), N, K, bits, _ptr(q), _ptr(s), _ptr(z)))
    return q, s, z


def unshard_host(gathered, G, B, widths):
    """hc_unshard_host: [G][B][Σw] gathered slices -> [B][G·Σw] canonical (uint16 bit patterns)."""
    widths = np.ascontiguousarray(widths, dtype=np.int32)
    gathered = np.ascontiguousarray(gathered, dtype=np.uint16)
    out = np.zeros((B, G * int(widths.sum())), dtype=np.uint16)
    check(lib().hc_unshard_host(_ptr(gathered), _ptr(out), G, B, len(widths), _ptr(widths)))
    return out


# ------------------------------------------------------------------ device context
class Context:
    """hc_ctx: owns the repacked weights of loaded windows on one CUDA device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().hc_create(C.byref(h), int(device)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            lib().hc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_layer(self, mats, stream=None):
        """mats: list of dicts with layer, window, slot, expert(-1), N, K, bits, group(128),
        codes, scales, zeros, U, V (numpy or torch), r_stored, r_alloc, row_begin(0), row_end(N), glue(0),
        factor_dtype(FACTORS_BF16; FACTORS_FP8: U / V e4m3 bytes + fp32 u_scale / v_scale [r_stored])."""
        arr = (_lib.hc_matrix_desc * len(mats))()
        for i, m in enumerate(mats):
            d = arr[i]
            d.layer, d.window_kind, d.slot = int(m["layer"]), int(m["window"]), int(m["slot"])
            d.expert = int(m.get("expert", -1))
            d.N, d.K, d.bits, d.group = int(m["N"]), int(m["K"]), int(m["bits"]), int(m.get("group", 128))
            d.codes, d.scales, d.zeros = _ptr(m["codes"]), _ptr(m["scales"]), _ptr(m["zeros"])
            d.U, d.V = _ptr(m.get("U")), _ptr(m.get("V"))
            d.r_stored, d.r_alloc = int(m.get("r_stored", 0)), int(m.get("r_alloc", 0))
            d.row_begin, d.row_end = int(m.get("row_begin", 0)), int(m.get("row_end", m["N"]))
            d.glue = int(m.get("glue", 0))
            d.factor_dtype = int(m.get("factor_dtype", 0))
            d.u_scale, d.v_scale = _ptr(m.get("u_scale")), _ptr(m.get("v_scale"))
        check(lib().hc_load_layer(self._h, arr, len(mats), _stream(stream)))

    def init_comm(self, rank: int, world: int, group=None):
        """Create the context's NCCL communicator: rank 0's unique id is broadcast through
        torch.distributed (any backend), then hc_set_comm."""
        import torch
        import torch.distributed as dist
        buf = np.zeros(128, dtype=np.uint8)
        if rank == 0:
            check(lib().hc_nccl_unique_id(buf.ctypes.data))
        obj = [buf.tobytes()]
        dist.broadcast_object_list(obj, src=0, group=group)
        buf = np.frombuffer(obj[0], dtype=np.uint8).copy()
        check(lib().hc_set_comm(self._h, buf.ctypes.data, int(rank), int(world)))

    def peer_region(self, world: int):
        """hc_peer_region: allocate this rank's peer region for the loaded shard; returns (base, bytes)."""
        base, nb = C.c_void_p(0), C.c_uint64(0)
        check(lib().hc_peer_region(self._h, int(world), C.addressof(base), C.addressof(nb)))
        return int(base.value), int(nb.value)

    def peer_set(self, rank: int, world: int, bases):
        """hc_peer_set: every rank's region base, already mapped in this process (in-process ranks)."""
        arr = (C.c_void_p * len(bases))(*[int(b) for b in bases])
        check(lib().hc_peer_set(self._h, int(rank), int(world), C.addressof(arr)))

    def init_peers(self, rank: int, world: int, group=None):
        """One process per GPU: allocate the peer region, exchange CUDA IPC handles through torch.distributed
        (any backend), hc_peer_connect."""
        import torch.distributed as dist
        self.peer_region(world)
        h = np.zeros(64, dtype=np.uint8)
        check(lib().hc_peer_ipc_handle(self._h, h.ctypes.data))
        allh = [None] * world
        dist.all_gather_object(allh, h.tobytes(), group=group)
        buf = np.frombuffer(b"".join(allh), dtype=np.uint8).copy()
        check(lib().hc_peer_connect(self._h, int(rank), int(world), buf.ctypes.data))

    def set_rank(self, layer, window, slot, r, expert=-1):
        check(lib().hc_set_rank(self._h, layer, window, slot, expert, r))

    def window_rows(self, layer, window, expert=-1) -> int:
        return int(lib().hc_window_rows(self._h, layer, window, expert))

    def stack_forward(self, x, y, B=None, stream=None):
        """hc_stack_forward: one decode step through all loaded layers (bf16 in, bf16 out)."""
        if B is None:
            B = x.shape[0]
        d = int(x.shape[-1])
        _check_buf("x", x, B * d, (2,), "bf16 [B, hidden]")
        _check_buf("y", y, B * d, (2,), "bf16 [B, hidden]")
        check(lib().hc_stack_forward(self._h, _ptr(x), int(B), _ptr(y), _stream(stream)))
        return y

    def moe_forward(self, layer, x, topk_idx, topk_gate, y, stream=None):
        """hc_moe_forward: grouped MoE expert layer.  x bf16 [T, K]; topk_idx int32 [T, k];
        topk_gate fp32 [T, k]; y fp32 [T, D] (device tensors or host arrays)."""
        T, k = int(topk_idx.shape[0]), int(topk_idx.shape[1])
        if not _is_int32(topk_idx):
            raise TypeError(f"topk_idx must be int32 (got {topk_idx.dtype}; e.g. torch.topk returns int64)")
        if not _is_f32(topk_gate):
            raise TypeError(f"topk_gate must be float32 (got {topk_gate.dtype})")
        _check_buf("topk_gate", topk_gate, T * k, (4,), "fp32 [T, k]")
        _check_buf("x", x, T * int(x.shape[-1]), (2,), "bf16 [T, K]")
        _check_buf("y", y, T, (4,), "fp32 [T, D]")
        check(lib().hc_moe_forward(self._h, int(layer), _ptr(x), T, _ptr(topk_idx), _ptr(topk_gate), k, _ptr(y),
                                   _stream(stream)))
        return y

    def moe_set_dynamic_ranks(self, layer, rtilde=None, k0=3):
        """hc_moe_set_dynamic_ranks: rtilde float [E, 3] (up, gate, down) or None (static ranks)."""
        if rtilde is None:
            check(lib().hc_moe_set_dynamic_ranks(self._h, int(layer), None, 0, int(k0)))
            return
        r = np.ascontiguousarray(rtilde, dtype=np.float32)
        check(lib().hc_moe_set_dynamic_ranks(self._h, int(layer), r.ctypes.data, int(r.shape[0]), int(k0)))

    def moe_last_ranks(self, T, topk):
        """hc_moe_last_ranks: int32 [T, topk, 3] ranks (up, gate, down) the device decided in the last
        hc_moe_forward with dynamic ranks (-1 for a skipped slot)."""
        out = np.zeros((int(T), int(topk), 3), dtype=np.int32)
        check(lib().hc_moe_last_ranks(self._h, out.ctypes.data, int(T), int(topk)))
        return out

    def calib_svd(self, W, codes, scales, zeros, bits, group, r, U, V, sigma=None, stream=None):
        """hc_calib_svd: device tensors W fp32 [M, N, K], canonical codes int32 [M, N, K*bits/32], scales bf16
        [M, N, K/g], zeros uint8 [M, N, K/g]; outputs float64 U [M, N, r], V [M, r, K], sigma [M, min(N, K)].
        Returns the number of Jacobi sweeps."""
        M, N, K = (int(v) for v in W.shape)
        sw = C.c_int32(0)
        check(lib().hc_calib_svd(self._h, _ptr(W), _ptr(codes), _ptr(scales), _ptr(zeros), M, N, K, int(bits),
                                 int(group), int(r), _ptr(U) if U is not None else None,
                                 _ptr(V) if V is not None else None, _ptr(sigma) if sigma is not None else None,
                                 C.addressof(sw), _stream(stream)))
        return int(sw.value)

    def calib_salience(self, sigma, phi, n_salient, tau=0.01, stream=None):
        """hc_calib_salience: device float64 sigma [M, n] -> phi float64 [M], n_salient int32 [M]."""
        M, n = (int(v) for v in sigma.shape)
        check(lib().hc_calib_salience(self._h, _ptr(sigma), M, n, float(tau), _ptr(phi), _ptr(n_salient), _stream(stream)))

    def compensated_linear(self, layer, window, x, y, B=None, expert=-1, out_dtype=OUT_F32, stream=None):
        """y[b, :] = concat_m ( deq(W_m)·x_b + U_m[:, :r_m]·(V_m[:r_m, :]·x_b) ).
        x: bf16 [B, K] (torch bf16 / uint16 bits, device or host); y: [B, rows] fp32 or bf16."""
        if B is None:
            B = x.shape[0]
        rows = self.window_rows(layer, window, expert)
        if rows < 0:
            raise HCError(HC_ERR_STATE, f"window ({layer},{window},{expert}) not loaded")
        _check_buf("x", x, B * int(x.shape[-1]), (2,), "bf16 [B, K]")
        _check_buf("y", y, B * rows, (4,) if out_dtype == OUT_F32 else (2,),
                   "fp32 [B, rows]" if out_dtype == OUT_F32 else "bf16 [B, rows]")
        check(lib().hc_compensated_linear(self._h, layer, window, expert, _ptr(x), int(B), _ptr(y),
                                          int(out_dtype), _stream(stream)))
        return y
