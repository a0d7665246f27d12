"""MicroMix (arXiv 2508.02343) hot path on B200 -- thin Python binding.

Argument marshalling only: every step of the path runs in the sm_100a kernels of
libmicromix_b200.so behind the C ABI in include/mm.h.  PyTorch provides device
memory and the current CUDA stream; there is no CPU fallback -- if the library
is missing or the device is not sm_100, calls raise.

Functions carry the C names:
    mm_plan_init, mm_calibrate_thresholds, mm_quantize_weight_offline,
    mm_reorder_quantize_act, mm_mixed_gemm_bf16, mm_reorder_act_bf16,
    mm_comm_init, mm_mixed_gemm_bf16_nshard_allgather,
    mm_mixed_gemm_bf16_nshard_peerstore (fused all-gather epilogue over peer memory).
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MM_LIB_PATH") or os.path.join(_HERE, "libmicromix_b200.so")   # override: tuning A/B builds

MM_E2M1, MM_E3M2, MM_E2M3, MM_E4M3, MM_E5M2 = range(5)
MM_SCALE_OCP, MM_SCALE_PAPER_EQ1 = 0, 1
STATUS = {0: "MM_OK", 1: "MM_ERR_INVALID_ARGUMENT", 2: "MM_ERR_SHAPE", 3: "MM_ERR_ALIGNMENT",
          4: "MM_ERR_PLAN_MISMATCH", 5: "MM_ERR_DEGENERATE", 6: "MM_ERR_UNSUPPORTED_DEVICE",
          7: "MM_ERR_CUDA", 8: "MM_ERR_NCCL", 9: "MM_ERR_WORKSPACE"}
SEG_BITS = (4, 6, 8)

# Every symbol include/mm.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "mm_padded_cols", "mm_code_pitch_bytes", "mm_codes_bytes", "mm_sf_bytes",
    "mm_calib_workspace_bytes", "mm_plan_init", "mm_calibrate_thresholds",
    "mm_quantize_weight_offline", "mm_reorder_quantize_act", "mm_mixed_gemm_bf16", "mm_gemm_workspace_bytes",
    "mm_peer_window_set_timeout", "mm_peer_window_error", "mm_gather_layout_words", "mm_plan_set_gather_layout",
    "mm_gather_layout_host", "mm_gather_wavefronts", "mm_mc_supported", "mm_mc_handle_bytes",
    "mm_mc_window_create", "mm_mc_window_bind", "mm_mc_window_local", "mm_mc_window_set_timeout",
    "mm_mc_window_error", "mm_mc_window_close", "mm_mc_barrier", "mm_mixed_gemm_bf16_nshard_nvls",
    "mm_reorder_act_bf16", "mm_set_gemm_config", "mm_launch_count", "mm_reset_launch_count",
    "mm_last_error", "mm_abi_version", "mm_nccl_unique_id_bytes", "mm_nccl_get_unique_id",
    "mm_comm_init", "mm_comm_destroy", "mm_mixed_gemm_bf16_nshard_allgather",
    "mm_calib_state_bytes", "mm_calib_accumulate", "mm_calib_finalize", "mm_plan_diagnostics",
    "mm_rmsnorm_reorder_quantize_act",
    "mm_peer_buffer_bytes", "mm_ipc_handle_bytes", "mm_ipc_get_handle", "mm_peer_window_open",
    "mm_peer_window_from_ptrs", "mm_peer_window_close", "mm_mixed_gemm_bf16_nshard_peerstore",
    "mm_peer_barrier",
]


class MMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class CPlan(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int32), ("n", ctypes.c_int32 * 3), ("fmt6", ctypes.c_int32),
                ("fmt8", ctypes.c_int32), ("rule", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("d_perm", ctypes.c_void_p), ("fingerprint", ctypes.c_uint64),
                ("tensor_max", ctypes.c_double), ("t4", ctypes.c_double), ("t6", ctypes.c_double),
                ("c", ctypes.c_int32 * 3), ("reserved2", ctypes.c_int32), ("d_layout", ctypes.c_void_p)]


class CDiag(ctypes.Structure):
    _fields_ = [("p", ctypes.c_double * 3), ("avg_bits", ctypes.c_double), ("stored_bytes_per_row", ctypes.c_int64),
                ("eq6_violations", ctypes.c_int32 * 2)]


class CMx(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("codes", ctypes.c_void_p * 3), ("sf", ctypes.c_void_p * 3),
                ("fingerprint", ctypes.c_uint64)]


_lib = None


def lib(build_if_missing: bool = False):
    """The loaded CUDA library; raises if it is not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            if build_if_missing:
                from .build import build
                build()
            else:
                raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                   "(python -m paper_2508_02343_b200.build)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        P, X = ctypes.POINTER(CPlan), ctypes.POINTER(CMx)
        sig = {
            "mm_padded_cols": (i64, [P, ctypes.c_int]),
            "mm_code_pitch_bytes": (i64, [P, ctypes.c_int]),
            "mm_codes_bytes": (i64, [P, i64, ctypes.c_int]),
            "mm_sf_bytes": (i64, [P, i64, ctypes.c_int]),
            "mm_calib_workspace_bytes": (i64, [i64, i32]),
            "mm_plan_init": (ctypes.c_int, [P, i32, ctypes.POINTER(i32), i32, i32, i32, vp, vp, vp]),
            "mm_calibrate_thresholds": (ctypes.c_int, [vp, i64, i32, i64, i32, i32, i32, vp, P, vp,
                                                       ctypes.c_size_t, vp, vp, vp]),
            "mm_quantize_weight_offline": (ctypes.c_int, [vp, i64, i64, P, X, vp]),
            "mm_reorder_quantize_act": (ctypes.c_int, [vp, i64, i64, P, X, vp]),
            "mm_mixed_gemm_bf16": (ctypes.c_int, [X, X, P, vp, i64, vp, ctypes.c_size_t, vp]),
            "mm_gemm_workspace_bytes": (i64, [P, i64, i64]),
            "mm_gather_layout_words": (i64, [i32]),
            "mm_plan_set_gather_layout": (ctypes.c_int, [P, vp, vp]),
            "mm_gather_layout_host": (ctypes.c_int, [i32, ctypes.POINTER(i32), vp, vp]),
            "mm_mc_supported": (i32, []),
            "mm_mc_handle_bytes": (i32, []),
            "mm_mc_window_create": (ctypes.c_int, [i32, i32, i64, i64, vp, ctypes.POINTER(vp)]),
            "mm_mc_window_bind": (ctypes.c_int, [vp]),
            "mm_mc_window_local": (vp, [vp]),
            "mm_mc_window_set_timeout": (ctypes.c_int, [vp, ctypes.c_double]),
            "mm_mc_window_error": (ctypes.c_int, [vp, ctypes.POINTER(i32)]),
            "mm_mc_window_close": (ctypes.c_int, [vp]),
            "mm_mc_barrier": (ctypes.c_int, [vp, vp]),
            "mm_mixed_gemm_bf16_nshard_nvls": (ctypes.c_int, [X, X, P, i64, vp, i32, vp]),
            "mm_gather_wavefronts": (i64, [i32, ctypes.POINTER(i32), vp, vp]),
            "mm_reorder_act_bf16": (ctypes.c_int, [vp, i64, i64, P, vp, i64, vp]),
            "mm_set_gemm_config": (ctypes.c_int, [i32, i32, i32]),
            "mm_launch_count": (i64, []),
            "mm_reset_launch_count": (None, []),
            "mm_last_error": (ctypes.c_char_p, []),
            "mm_abi_version": (i32, []),
            "mm_nccl_unique_id_bytes": (i32, []),
            "mm_nccl_get_unique_id": (ctypes.c_int, [vp]),
            "mm_comm_init": (ctypes.c_int, [i32, i32, vp, ctypes.POINTER(vp)]),
            "mm_comm_destroy": (ctypes.c_int, [vp]),
            "mm_mixed_gemm_bf16_nshard_allgather": (ctypes.c_int, [X, X, P, i64, vp, i64, vp, ctypes.c_size_t,
                                                                   vp, vp]),
            "mm_calib_state_bytes": (i64, [i32]),
            "mm_calib_accumulate": (ctypes.c_int, [vp, i64, i32, i64, vp, ctypes.c_size_t, vp, vp]),
            "mm_calib_finalize": (ctypes.c_int, [vp, i32, i32, i32, i32, vp, P, vp, vp, vp, vp]),
            "mm_plan_diagnostics": (ctypes.c_int, [P, vp, vp, ctypes.POINTER(CDiag)]),
            "mm_rmsnorm_reorder_quantize_act": (ctypes.c_int, [vp, i64, i64, vp, ctypes.c_double, P, X, vp]),
            "mm_peer_buffer_bytes": (ctypes.c_size_t, [i64, i64]),
            "mm_ipc_handle_bytes": (i32, []),
            "mm_ipc_get_handle": (ctypes.c_int, [vp, vp]),
            "mm_peer_window_open": (ctypes.c_int, [i32, i32, vp, vp, i64, i64, ctypes.POINTER(vp)]),
            "mm_peer_window_from_ptrs": (ctypes.c_int, [i32, i32, ctypes.POINTER(vp), i64, i64, ctypes.POINTER(vp)]),
            "mm_peer_window_close": (ctypes.c_int, [vp]),
            "mm_mixed_gemm_bf16_nshard_peerstore": (ctypes.c_int, [X, X, P, i64, vp, i32, vp]),
            "mm_peer_barrier": (ctypes.c_int, [vp, vp]),
            "mm_peer_window_set_timeout": (ctypes.c_int, [vp, ctypes.c_double]),
            "mm_peer_window_error": (ctypes.c_int, [vp, ctypes.POINTER(i32)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise MMError(st, lib().mm_last_error().decode())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else ctypes.c_void_p(0)


class Plan:
    """A channel plan (include/mm.h mm_plan) plus the device permutation it borrows."""

    def __init__(self, c: CPlan, d_perm: torch.Tensor, layout: bool | None = None):
        self.c = c
        self.d_perm = d_perm
        self.d_layout = None
        if layout is None:
            layout = os.environ.get("MM_NO_GATHER_LAYOUT", "0") != "1"
        if layout:
            self.set_gather_layout()

    def set_gather_layout(self, stream=None):
        """Attach the plan-time gather layout (mm_plan_set_gather_layout; offline, synchronizes)."""
        words = int(lib().mm_gather_layout_words(self.c.K))
        buf = torch.empty(max(words, 4), dtype=torch.int32, device=self.d_perm.device)
        _check(lib().mm_plan_set_gather_layout(ctypes.byref(self.c), _ptr(buf), _stream(stream)))
        self.d_layout = buf

    @property
    def K(self):
        return self.c.K

    @property
    def n(self):
        return tuple(self.c.n)

    @property
    def fmt6(self):
        return self.c.fmt6

    @property
    def fmt8(self):
        return self.c.fmt8

    @property
    def rule(self):
        return self.c.rule

    def padded_cols(self, g):
        return lib().mm_padded_cols(ctypes.byref(self.c), g)

    def pitch(self, g):
        return lib().mm_code_pitch_bytes(ctypes.byref(self.c), g)

    def codes_bytes(self, rows, g):
        return lib().mm_codes_bytes(ctypes.byref(self.c), rows, g)

    def sf_bytes(self, rows, g):
        return lib().mm_sf_bytes(ctypes.byref(self.c), rows, g)

    def perm_host(self):
        return self.d_perm.cpu()


class MXTensor:
    """A quantized operand: per-segment packed codes and E8M0 scale atoms (uint8 buffers)."""

    def __init__(self, plan: Plan, rows: int, device=None):
        device = device or plan.d_perm.device
        self.plan = plan
        self.rows = rows
        self.codes, self.sf = [], []
        c = CMx()
        c.rows = rows
        for g in range(3):
            if plan.n[g] == 0:
                self.codes.append(None)
                self.sf.append(None)
                continue
            cb = torch.empty(max(plan.codes_bytes(rows, g), 1), dtype=torch.uint8, device=device)
            sb = torch.empty(max(plan.sf_bytes(rows, g), 1), dtype=torch.uint8, device=device)
            self.codes.append(cb)
            self.sf.append(sb)
            c.codes[g] = cb.data_ptr()
            c.sf[g] = sb.data_ptr()
        self.c = c

    def codes2d(self, g):
        return self.codes[g][: self.plan.codes_bytes(self.rows, g)].view(self.rows, self.plan.pitch(g))


def mm_plan_init(K, n, perm, fmt6=MM_E3M2, fmt8=MM_E4M3, rule=MM_SCALE_OCP, device="cuda") -> Plan:
    perm = torch.as_tensor(perm, dtype=torch.int32).contiguous().cpu()
    d_perm = torch.empty(K, dtype=torch.int32, device=device)
    c = CPlan()
    nn = (ctypes.c_int32 * 3)(*[int(v) for v in n])
    _check(lib().mm_plan_init(ctypes.byref(c), K, nn, fmt6, fmt8, rule, ctypes.c_void_p(perm.data_ptr()),
                              _ptr(d_perm), _stream()))
    return Plan(c, d_perm)


def mm_calibrate_thresholds(x: torch.Tensor, fmt6=MM_E3M2, fmt8=MM_E4M3, rule=MM_SCALE_OCP,
                            return_stats=False):
    assert x.dtype == torch.bfloat16 and x.dim() == 2 and x.stride(1) == 1
    L, K = x.shape
    d_perm = torch.empty(K, dtype=torch.int32, device=x.device)
    ws = torch.empty(max(lib().mm_calib_workspace_bytes(L, K), 1), dtype=torch.uint8, device=x.device)
    chmax = torch.empty(K, dtype=torch.float64)
    chmean = torch.empty(K, dtype=torch.float64)
    c = CPlan()
    _check(lib().mm_calibrate_thresholds(_ptr(x), L, K, x.stride(0), fmt6, fmt8, rule, _ptr(d_perm),
                                         ctypes.byref(c), _ptr(ws), ws.numel(),
                                         ctypes.c_void_p(chmax.data_ptr()), ctypes.c_void_p(chmean.data_ptr()),
                                         _stream()))
    plan = Plan(c, d_perm)
    return (plan, chmax, chmean) if return_stats else plan


class CalibState:
    """Streaming calibration (include/mm.h mm_calib_*): accumulate batches, then finalize."""

    def __init__(self, K: int, device="cuda"):
        self.K = K
        self.buf = torch.zeros(lib().mm_calib_state_bytes(K), dtype=torch.uint8, device=device)

    def accumulate(self, x: torch.Tensor):
        assert x.dtype == torch.bfloat16 and x.dim() == 2 and x.stride(1) == 1 and x.shape[1] == self.K
        L = x.shape[0]
        ws = torch.empty(max(lib().mm_calib_workspace_bytes(L, self.K), 1), dtype=torch.uint8, device=x.device)
        _check(lib().mm_calib_accumulate(_ptr(x), L, self.K, x.stride(0), _ptr(ws), ws.numel(), _ptr(self.buf),
                                         _stream()))
        self._ws = ws   # keep alive until the queued work ran
        return self

    def finalize(self, fmt6=MM_E3M2, fmt8=MM_E4M3, rule=MM_SCALE_OCP, return_stats=False):
        d_perm = torch.empty(self.K, dtype=torch.int32, device=self.buf.device)
        chmax = torch.empty(self.K, dtype=torch.float64)
        chmean = torch.empty(self.K, dtype=torch.float64)
        rows = ctypes.c_int64(0)
        c = CPlan()
        _check(lib().mm_calib_finalize(_ptr(self.buf), self.K, fmt6, fmt8, rule, _ptr(d_perm), ctypes.byref(c),
                                       ctypes.c_void_p(chmax.data_ptr()), ctypes.c_void_p(chmean.data_ptr()),
                                       ctypes.byref(rows), _stream()))
        plan = Plan(c, d_perm)
        return (plan, chmax, chmean, rows.value) if return_stats else plan


def mm_plan_diagnostics(plan: Plan, chmax=None) -> dict:
    """p4/p6/p8, average bits (Table 1 accounting), stored bytes per row, Eq. 6 violations."""
    d = CDiag()
    perm = plan.perm_host().contiguous() if chmax is not None else None
    cm = torch.as_tensor(chmax, dtype=torch.float64).contiguous() if chmax is not None else None
    _check(lib().mm_plan_diagnostics(ctypes.byref(plan.c), ctypes.c_void_p(cm.data_ptr()) if cm is not None else None,
                                     ctypes.c_void_p(perm.data_ptr()) if perm is not None else None, ctypes.byref(d)))
    return {"p": tuple(d.p), "avg_bits": d.avg_bits, "stored_bytes_per_row": d.stored_bytes_per_row,
            "eq6_violations": tuple(d.eq6_violations)}


def _rq(fn, x: torch.Tensor, plan: Plan, out: MXTensor | None, stream=None) -> MXTensor:
    assert x.dtype == torch.bfloat16 and x.dim() == 2 and x.stride(1) == 1
    rows = x.shape[0]
    if out is None:
        out = MXTensor(plan, rows, x.device)
    _check(fn(_ptr(x), rows, x.stride(0), ctypes.byref(plan.c), ctypes.byref(out.c), _stream(stream)))
    return out


def mm_quantize_weight_offline(w: torch.Tensor, plan: Plan, out: MXTensor | None = None, stream=None):
    return _rq(lib().mm_quantize_weight_offline, w, plan, out, stream)


def mm_reorder_quantize_act(x: torch.Tensor, plan: Plan, out: MXTensor | None = None, stream=None):
    return _rq(lib().mm_reorder_quantize_act, x, plan, out, stream)


def mm_rmsnorm_reorder_quantize_act(x: torch.Tensor, gamma: torch.Tensor, eps: float, plan: Plan,
                                    out: MXTensor | None = None, stream=None) -> MXTensor:
    """RMSNorm(x) * gamma, reordered and quantized in one kernel (F2 fusion)."""
    assert x.dtype == torch.bfloat16 and x.dim() == 2 and x.stride(1) == 1
    assert gamma.dtype == torch.bfloat16 and gamma.is_contiguous() and gamma.numel() == x.shape[1]
    rows = x.shape[0]
    if out is None:
        out = MXTensor(plan, rows, x.device)
    _check(lib().mm_rmsnorm_reorder_quantize_act(_ptr(x), rows, x.stride(0), _ptr(gamma), float(eps),
                                                 ctypes.byref(plan.c), ctypes.byref(out.c), _stream(stream)))
    return out


def mm_gemm_workspace_bytes(plan: Plan, M: int, N: int) -> int:
    n = int(lib().mm_gemm_workspace_bytes(ctypes.byref(plan.c), M, N))
    if n < 0:
        raise MMError(1, "mm_gemm_workspace_bytes: invalid arguments")
    return n


_WS = {}   # (device index, stream handle) -> zero-filled uint8 workspace (grown, never shrunk)


def gemm_workspace(plan: Plan, M: int, N: int, stream=None) -> torch.Tensor | None:
    """The caller-owned GEMM workspace (include/mm.h) this binding keeps per (device,
    stream): allocated by torch, zero-filled once, grown when a larger one is needed.
    Call it once before capturing a CUDA graph so the capture allocates nothing."""
    need = mm_gemm_workspace_bytes(plan, M, N)
    if need == 0:
        return None
    dev = plan.d_perm.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    key = (dev.index, int(s.cuda_stream))
    ws = _WS.get(key)
    if ws is None or ws.numel() < need:
        if ws is not None:
            s.synchronize()    # the old buffer may still be in use by queued work
        ws = torch.zeros(need, dtype=torch.uint8, device=dev)
        torch.cuda.current_stream(dev).synchronize()
        _WS[key] = ws
    return ws


def mm_mixed_gemm_bf16(a: MXTensor, w: MXTensor, plan: Plan, out: torch.Tensor | None = None,
                       stream=None, workspace: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(a.rows, w.rows, dtype=torch.bfloat16, device=plan.d_perm.device)
    assert out.dtype == torch.bfloat16 and out.stride(1) == 1
    ws = workspace if workspace is not None else gemm_workspace(plan, a.rows, w.rows, stream)
    _check(lib().mm_mixed_gemm_bf16(ctypes.byref(a.c), ctypes.byref(w.c), ctypes.byref(plan.c), _ptr(out),
                                    out.stride(0), None if ws is None else _ptr(ws),
                                    0 if ws is None else ws.numel(), _stream(stream)))
    return out


def mm_reorder_act_bf16(x: torch.Tensor, plan: Plan) -> torch.Tensor:
    out = torch.empty_like(x)
    _check(lib().mm_reorder_act_bf16(_ptr(x), x.shape[0], x.stride(0), ctypes.byref(plan.c), _ptr(out),
                                     out.stride(0), _stream()))
    return out


def mm_set_gemm_config(block_n=0, num_stages=0, max_ctas=0):
    _check(lib().mm_set_gemm_config(block_n, num_stages, max_ctas))


def launch_count() -> int:
    return lib().mm_launch_count()


def reset_launch_count():
    lib().mm_reset_launch_count()


# ---- multi-GPU -------------------------------------------------------------------
def nccl_unique_id() -> bytes:
    n = lib().mm_nccl_unique_id_bytes()
    buf = ctypes.create_string_buffer(n)
    _check(lib().mm_nccl_get_unique_id(buf))
    return buf.raw


def mm_comm_init(rank: int, world: int, unique_id: bytes):
    buf = ctypes.create_string_buffer(unique_id, len(unique_id))
    comm = ctypes.c_void_p()
    _check(lib().mm_comm_init(rank, world, buf, ctypes.byref(comm)))
    return comm


def mm_comm_destroy(comm):
    _check(lib().mm_comm_destroy(comm))


def mm_mixed_gemm_bf16_nshard_allgather(a: MXTensor, w_shard: MXTensor, plan: Plan, n_total: int, comm,
                                        out: torch.Tensor | None = None, stage: torch.Tensor | None = None,
                                        stream=None):
    dev = plan.d_perm.device
    if out is None:
        out = torch.empty(a.rows, n_total, dtype=torch.bfloat16, device=dev)
    if stage is None:
        stage = torch.empty(a.rows * n_total, dtype=torch.bfloat16, device=dev)
    _check(lib().mm_mixed_gemm_bf16_nshard_allgather(ctypes.byref(a.c), ctypes.byref(w_shard.c),
                                                     ctypes.byref(plan.c), n_total, _ptr(out), out.stride(0),
                                                     _ptr(stage), stage.numel() * stage.element_size(), comm,
                                                     _stream(stream)))
    return out


def shard_rows(N: int, world: int, rank: int):
    """Rows of W owned by `rank` under N-sharding (host logic, CPU-testable)."""
    from .dist import shard_rows as _sr
    return _sr(N, world, rank)


# ---- fused GEMM + all-gather epilogue over peer memory (NEXT F1) ------------------
def mm_peer_buffer_bytes(M: int, ldy: int) -> int:
    return int(lib().mm_peer_buffer_bytes(M, ldy))


def peer_buffer(M: int, ldy: int, device=None) -> torch.Tensor:
    """A zero-filled peer buffer ([Y: BF16 M x ldy][flags]) as a uint8 tensor (256-B
    aligned: the caching allocator aligns to 512 B)."""
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    return torch.zeros(mm_peer_buffer_bytes(M, ldy), dtype=torch.uint8, device=dev)


def peer_y(buf: torch.Tensor, M: int, ldy: int) -> torch.Tensor:
    """The BF16 [M, ldy] Y view of a peer buffer."""
    return buf[: M * ldy * 2].view(torch.bfloat16).view(M, ldy)


def ipc_handle(buf: torch.Tensor) -> bytes:
    n = lib().mm_ipc_handle_bytes()
    out = ctypes.create_string_buffer(n)
    _check(lib().mm_ipc_get_handle(_ptr(buf), out))
    return out.raw


class PeerWindow:
    """This rank's table of every rank's peer buffer (include/mm.h)."""

    def __init__(self, handle, rank: int, world: int, M: int, ldy: int, keep=()):
        self.h, self.rank, self.world, self.M, self.ldy = handle, rank, world, M, ldy
        self._keep = keep   # buffers that must outlive the window

    @classmethod
    def open(cls, rank: int, world: int, local_buf: torch.Tensor, handles: list, M: int, ldy: int):
        blob = b"".join(handles)
        cbuf = ctypes.create_string_buffer(blob, len(blob))
        h = ctypes.c_void_p()
        _check(lib().mm_peer_window_open(rank, world, _ptr(local_buf), cbuf, M, ldy, ctypes.byref(h)))
        return cls(h, rank, world, M, ldy, (local_buf,))

    @classmethod
    def from_ptrs(cls, rank: int, world: int, bufs: list, M: int, ldy: int):
        arr = (ctypes.c_void_p * world)(*[b.data_ptr() for b in bufs])
        h = ctypes.c_void_p()
        _check(lib().mm_peer_window_from_ptrs(rank, world, arr, M, ldy, ctypes.byref(h)))
        return cls(h, rank, world, M, ldy, tuple(bufs))

    def close(self):
        if self.h is not None:
            _check(lib().mm_peer_window_close(self.h))
            self.h = None

    def set_timeout(self, seconds: float):
        """Barrier timeout (0 = wait forever, the default)."""
        _check(lib().mm_peer_window_set_timeout(self.h, float(seconds)))

    def error(self) -> int:
        """Rank a timed-out barrier waited for, or -1 (synchronous read)."""
        v = ctypes.c_int32()
        _check(lib().mm_peer_window_error(self.h, ctypes.byref(v)))
        return v.value


def mm_mixed_gemm_bf16_nshard_peerstore(a: MXTensor, w_shard: MXTensor, plan: Plan, n_total: int,
                                        win: PeerWindow, barrier: bool = True, stream=None):
    _check(lib().mm_mixed_gemm_bf16_nshard_peerstore(ctypes.byref(a.c), ctypes.byref(w_shard.c),
                                                     ctypes.byref(plan.c), n_total, win.h, int(barrier),
                                                     _stream(stream)))


def mm_peer_barrier(win: PeerWindow, stream=None):
    _check(lib().mm_peer_barrier(win.h, _stream(stream)))


# ---- fused all-gather over NVLS (multicast; include/mm.h) ---------------------------
def mc_supported() -> bool:
    return bool(lib().mm_mc_supported())


class McWindow:
    """This rank's view of a multicast object spanning every rank's [Y][flags] buffer.
    create() is collective over the torch process group (world 1 without one)."""

    def __init__(self, h, rank, world, M, ldy):
        self.h, self.rank, self.world, self.M, self.ldy = h, rank, world, M, ldy

    @classmethod
    def create(cls, M: int, ldy: int, group=None):
        import torch.distributed as dist
        dist_on = dist.is_available() and dist.is_initialized()
        rank = dist.get_rank(group) if dist_on else 0
        world = dist.get_world_size(group) if dist_on else 1
        rec = ctypes.create_string_buffer(lib().mm_mc_handle_bytes())
        h = ctypes.c_void_p()
        err = ""

        def agree(ok: bool):
            """Every rank learns whether all ranks succeeded (no rank is left waiting)."""
            if world == 1:
                return ok
            t = torch.tensor([1 if ok else 0], dtype=torch.int32,
                             device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            return bool(t.item())

        st = lib().mm_mc_window_create(0, world, M, ldy, rec, ctypes.byref(h)) if rank == 0 else 0
        if st != 0:
            err = lib().mm_last_error().decode()
        if world > 1:
            obj = [rec.raw if (rank == 0 and st == 0) else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            if rank != 0 and obj[0] is not None:
                rec = ctypes.create_string_buffer(obj[0], len(obj[0]))
                st = lib().mm_mc_window_create(rank, world, M, ldy, rec, ctypes.byref(h))
                if st != 0:
                    err = lib().mm_last_error().decode()
            elif rank != 0:
                st, err = 7, "rank 0 could not create the multicast object"
        if not agree(st == 0):                  # every device added before any bind
            if h.value:
                lib().mm_mc_window_close(h)
            raise MMError(7, "multicast window: " + (err or "another rank failed"))
        st = lib().mm_mc_window_bind(h)
        err = "" if st == 0 else lib().mm_last_error().decode()
        if not agree(st == 0):                  # every buffer bound and zeroed before use
            lib().mm_mc_window_close(h)
            raise MMError(7, "multicast window bind: " + (err or "another rank failed"))
        return cls(h, rank, world, M, ldy)

    def y(self) -> torch.Tensor:
        """This rank's Y [M, ldy] (BF16) as a torch view of the window's local buffer."""
        ptr = lib().mm_mc_window_local(self.h)
        n = self.M * self.ldy
        return _from_ptr(ptr, n, torch.bfloat16).view(self.M, self.ldy)

    def set_timeout(self, seconds: float):
        _check(lib().mm_mc_window_set_timeout(self.h, float(seconds)))

    def timed_out(self) -> bool:
        v = ctypes.c_int32()
        _check(lib().mm_mc_window_error(self.h, ctypes.byref(v)))
        return bool(v.value)

    def close(self):
        if self.h is not None:
            _check(lib().mm_mc_window_close(self.h))
            self.h = None


def _from_ptr(ptr: int, numel: int, dtype) -> torch.Tensor:
    """A torch tensor over device memory the library owns (no copy; valid while it lives)."""
    class _Cai:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (numel,), "typestr": "<i2", "data": (ptr, False),
                                             "version": 3, "strides": None}
    return torch.as_tensor(_Cai(), device="cuda").view(dtype)


def mm_mixed_gemm_bf16_nshard_nvls(a: MXTensor, w_shard: MXTensor, plan: Plan, n_total: int, win: McWindow,
                                   barrier: bool = True, stream=None):
    _check(lib().mm_mixed_gemm_bf16_nshard_nvls(ctypes.byref(a.c), ctypes.byref(w_shard.c), ctypes.byref(plan.c),
                                                n_total, win.h, int(barrier), _stream(stream)))


def mm_mc_barrier(win: McWindow, stream=None):
    _check(lib().mm_mc_barrier(win.h, _stream(stream)))
