"""CPU checks of the C ABI: the library builds/loads and exports every symbol
include/mm.h declares; size queries and host-side validation (no GPU needed)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

import paper_2508_02343_b200 as mm


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "mm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = set(re.findall(r"\b(mm_[a-z0-9_]+)\s*\(", txt))
    return sorted(names)


@pytest.fixture(scope="module")
def L():
    from paper_2508_02343_b200.build import build
    build()
    return mm.lib()


def test_header_matches_binding_list():
    assert sorted(mm.EXPORTS) == _header_symbols()


def test_library_exports_every_symbol(L):
    for name in _header_symbols():
        assert hasattr(L, name), name
    assert L.mm_abi_version() == 3


def _plan(K, n, fmt6=mm.MM_E3M2, fmt8=mm.MM_E4M3):
    c = mm.CPlan()
    c.K = K
    for i in range(3):
        c.n[i] = n[i]
    c.fmt6, c.fmt8 = fmt6, fmt8
    return c


def test_size_queries(L):
    c = _plan(4096, (2240, 1184, 672))
    p = ctypes.byref(c)
    assert [L.mm_padded_cols(p, g) for g in range(3)] == [2304, 1280, 768]
    assert [L.mm_code_pitch_bytes(p, g) for g in range(3)] == [1152, 960, 768]
    assert L.mm_codes_bytes(p, 2048, 1) == 2048 * 960
    assert L.mm_sf_bytes(p, 2000, 0) == 2048 * 2304 // 32
    assert L.mm_sf_bytes(p, 16, 2) == 128 * 768 // 32
    assert L.mm_padded_cols(p, 3) == -1
    assert L.mm_calib_workspace_bytes(16384, 4096) > 0


def test_plan_init_validation_on_host(L):
    c = mm.CPlan()
    n = (ctypes.c_int32 * 3)(64, 32, 32)
    perm = (ctypes.c_int32 * 128)(*([0] * 128))     # not a bijection
    st = L.mm_plan_init(ctypes.byref(c), 128, n, mm.MM_E3M2, mm.MM_E4M3, 0, perm, ctypes.c_void_p(16), None)
    assert st == 1 and b"bijection" in L.mm_last_error()
    bad_n = (ctypes.c_int32 * 3)(64, 30, 34)
    st = L.mm_plan_init(ctypes.byref(c), 128, bad_n, mm.MM_E3M2, mm.MM_E4M3, 0, perm, ctypes.c_void_p(16), None)
    assert st == 2
    st = L.mm_plan_init(ctypes.byref(c), 128, n, mm.MM_E4M3, mm.MM_E4M3, 0, perm, ctypes.c_void_p(16), None)
    assert st == 1


def test_calls_fail_loudly_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = _plan(128, (64, 32, 32))
    x = mm.CMx()
    st = L.mm_reorder_quantize_act(ctypes.c_void_p(0), 4, 128, ctypes.byref(c), ctypes.byref(x), None)
    assert st != 0


def test_shard_rows_host_logic():
    assert mm.shard_rows(8192, 8, 3) == (3072, 4096)
    with pytest.raises(ValueError):
        mm.shard_rows(100, 8, 0)


def test_plan_diagnostics_host(L):
    """mm_plan_diagnostics is host-only: p, Table-1 average bits, stored bytes per row
    and Eq. 6 violations against the oracle's own accounting."""
    import numpy as np
    from oracle import calib as ocal
    from synth import bf16_bits, gen_act
    K = 512
    cal = ocal.calibrate(bf16_bits(gen_act(300, K, 1000, 2000)))
    c = _plan(K, cal["n"])
    c.t4, c.t6 = cal["t4"], cal["t6"]
    chmax = np.ascontiguousarray(cal["chmax"], dtype=np.float64)
    perm = np.ascontiguousarray(cal["perm"], dtype=np.int32)
    d = mm.CDiag()
    st = L.mm_plan_diagnostics(ctypes.byref(c), ctypes.c_void_p(chmax.ctypes.data), ctypes.c_void_p(perm.ctypes.data),
                               ctypes.byref(d))
    assert st == 0
    assert abs(d.avg_bits - ocal.avg_bits(cal["n"])) < 1e-12
    assert tuple(d.eq6_violations) == ocal.eq6_violations(cal["perm"], cal["n"], cal["chmax"], cal["t4"], cal["t6"])
    assert [round(v * K) for v in d.p] == list(cal["n"])
    pitch = [(n + 127) // 128 * 128 * b // 8 for n, b in zip(cal["n"], (4, 6, 8))]
    assert d.stored_bytes_per_row == sum(pitch) + sum((n + 127) // 128 * 4 for n in cal["n"])


def test_peer_window_host_queries_and_validation(L):
    """Fused all-gather epilogue (NEXT F1): buffer size, handle size and the window
    argument checks are host logic."""
    # [Y: BF16 M x ldy padded to 256 B][64 x u32 flags]
    assert L.mm_peer_buffer_bytes(3, 8) == 256 + 256
    assert L.mm_peer_buffer_bytes(2048, 8192) == 2048 * 8192 * 2 + 256
    assert L.mm_ipc_handle_bytes() == 72            # cudaIpcMemHandle_t + u64 offset
    h = ctypes.c_void_p()
    bufs = (ctypes.c_void_p * 9)(*([256] * 9))
    assert L.mm_peer_window_from_ptrs(0, 9, bufs, 16, 64, ctypes.byref(h)) == 1      # world > 8
    assert L.mm_peer_window_from_ptrs(3, 2, bufs, 16, 64, ctypes.byref(h)) == 1      # rank >= world
    assert L.mm_peer_window_from_ptrs(0, 2, bufs, 16, 60, ctypes.byref(h)) == 2      # ldy % 8
    odd = (ctypes.c_void_p * 2)(256, 257)
    assert L.mm_peer_window_from_ptrs(0, 2, odd, 16, 64, ctypes.byref(h)) == 3       # alignment
    assert L.mm_peer_window_from_ptrs(1, 2, bufs, 16, 64, ctypes.byref(h)) == 0
    assert L.mm_peer_window_close(h) == 0
    assert L.mm_peer_window_close(None) == 0


def test_gemm_config_values(L):
    for bn in (0, 1, 128, 256, 512):
        assert L.mm_set_gemm_config(bn, 0, 0) == 0
    assert L.mm_set_gemm_config(64, 0, 0) == 1
    assert L.mm_set_gemm_config(0, 0, 0) == 0


def test_gather_layout_host(L):
    """The plan-time gather layout (layout.cpp): per 32-channel line a
    parity-preserving permutation of the eight 4-channel chunks, with fewer gather bank
    wavefronts than the natural layout for a calibrated-like permutation."""
    import numpy as np
    K, n = 4096, (2240, 1184, 672)
    perm = np.random.default_rng(3).permutation(K).astype(np.int32)
    nn = (ctypes.c_int32 * 3)(*n)
    lay = np.zeros(K // 32, dtype=np.uint32)
    assert L.mm_gather_layout_host(K, nn, perm.ctypes.data, lay.ctypes.data) == 0
    for w in lay:
        pos = [(int(w) >> (4 * c)) & 15 for c in range(8)]
        assert sorted(pos) == list(range(8))
        assert all(pos[c] % 2 == c % 2 for c in range(8))
    nat = L.mm_gather_wavefronts(K, nn, perm.ctypes.data, None)
    opt = L.mm_gather_wavefronts(K, nn, perm.ctypes.data, lay.ctypes.data)
    assert 0 < opt <= 0.85 * nat, (nat, opt)
    assert L.mm_gather_layout_host(K + 1, nn, perm.ctypes.data, lay.ctypes.data) == 1
