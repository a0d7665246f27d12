"""GPU checks of the boundary contract of include/mm.h: the hot calls
allocate nothing and never synchronize -- the small-M split-K partials are reduced
inside a thread-block cluster, the opt-in stream-K partials live in a caller
workspace sized by mm_gemm_workspace_bytes -- so the small-M (decode) path can be
captured into a CUDA graph; errors are reported before any
launch; a peer barrier whose peer never arrives reports instead of trapping."""
import numpy as np
import pytest
import torch

import paper_2508_02343_b200 as mm
from oracle import gemm as ogemm
from synth import bf16_bits, gen_act, gen_perm, gen_weight

pytestmark = pytest.mark.gpu


def _ops(M, N, n, seed=51):
    K = sum(n)
    plan = mm.mm_plan_init(K, n, gen_perm(K, seed))
    a = mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2001).cuda(), plan)
    w = mm.mm_quantize_weight_offline(gen_weight(N, K, 3000).cuda(), plan)
    return plan, a, w


def test_workspace_query_matches_paths(monkeypatch):
    plan, _, _ = _ops(16, 4096, (2240, 1184, 672))
    assert mm.mm_gemm_workspace_bytes(plan, 16, 4096) == 0       # small-M split-K: reduced in a cluster (DSMEM)
    assert mm.mm_gemm_workspace_bytes(plan, 2048, 4096) == 0     # CTA-pair tiles
    assert mm.mm_gemm_workspace_bytes(plan, 0, 4096) == 0
    monkeypatch.setenv("MM_GEMM_STREAMK", "1")                  # stream-K: 80 tiles on 74 pairs -> partials
    assert mm.mm_gemm_workspace_bytes(plan, 2048, 2560) > 0


def test_workspace_too_small_is_an_error_and_enqueues_nothing(monkeypatch):
    monkeypatch.setenv("MM_GEMM_STREAMK", "1")
    plan, a, w = _ops(2048, 2560, (2240, 1184, 672))
    need = mm.mm_gemm_workspace_bytes(plan, 2048, 2560)
    assert need > 0
    ws = torch.zeros(need - 256, dtype=torch.uint8, device="cuda")
    y = torch.full((2048, 2560), 7.0, dtype=torch.bfloat16, device="cuda")
    n0 = mm.launch_count()
    with pytest.raises(mm.MMError) as e:
        mm.mm_mixed_gemm_bf16(a, w, plan, out=y, workspace=ws)
    assert e.value.status == 9
    assert mm.launch_count() == n0
    torch.cuda.synchronize()
    assert bool((y == 7.0).all())


@pytest.mark.parametrize("M", [1, 16, 64])
def test_small_m_gemm_captured_in_cuda_graph(M):
    """Decode-like M: RQ + split-K GEMM captured once, replayed with new inputs; equal
    to eager execution bit for bit and within the oracle bar."""
    N, n = 4096, (2240, 1184, 672)
    K = sum(n)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 52))
    wq = mm.mm_quantize_weight_offline(gen_weight(N, K, 3000).cuda(), plan)
    x_static = gen_act(M, K, 1000, 2100).cuda()
    s = torch.cuda.Stream()
    ws = mm.gemm_workspace(plan, M, N, stream=s)          # (none needed: cluster split-K reduction)
    a = mm.MXTensor(plan, M, x_static.device)
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):                             # warm-up (attributes, tensor maps)
        mm.mm_reorder_quantize_act(x_static, plan, out=a, stream=s)
        mm.mm_mixed_gemm_bf16(a, wq, plan, out=y, stream=s, workspace=ws)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        mm.mm_reorder_quantize_act(x_static, plan, out=a, stream=s)
        mm.mm_mixed_gemm_bf16(a, wq, plan, out=y, stream=s, workspace=ws)
    for seed in (2101, 2102):
        x = gen_act(M, K, 1000, seed)
        x_static.copy_(x.cuda())
        g.replay()
        torch.cuda.synchronize()
        y_eager = mm.mm_mixed_gemm_bf16(mm.mm_reorder_quantize_act(x.cuda(), plan), wq, plan)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), y_eager.view(torch.int16)), seed
        yref, _ = ogemm.mixed_linear_ref(bf16_bits(x), bf16_bits(gen_weight(N, K, 3000)),
                                         plan.perm_host().numpy(), plan.n)
        assert ogemm.rel_fro(y.double().cpu().numpy(), yref) <= 2e-3


def test_nshard_allgather_rejects_bad_y_before_launch():
    plan, a, w = _ops(32, 256, (128, 64, 64))
    comm = mm.mm_comm_init(0, 1, mm.nccl_unique_id())
    try:
        n0 = mm.launch_count()
        stage = torch.empty(32 * 256, dtype=torch.bfloat16, device="cuda")
        L = mm.lib()
        import ctypes
        st = L.mm_mixed_gemm_bf16_nshard_allgather(ctypes.byref(a.c), ctypes.byref(w.c), ctypes.byref(plan.c), 256,
                                                   None, 256, stage.data_ptr(), stage.numel() * 2, comm, None)
        assert st == 3                                      # Y NULL -> alignment error
        y = torch.empty(32, 256, dtype=torch.bfloat16, device="cuda")
        st = L.mm_mixed_gemm_bf16_nshard_allgather(ctypes.byref(a.c), ctypes.byref(w.c), ctypes.byref(plan.c), 256,
                                                   y.data_ptr(), 256, stage.data_ptr(), 100, comm, None)
        assert st == 9                                      # stage too small
        assert mm.launch_count() == n0
    finally:
        mm.mm_comm_destroy(comm)


def test_peer_barrier_timeout_reports_missing_rank():
    """Two virtual ranks; only rank 0 reaches the barrier.  With a 0.2 s timeout its
    barrier gives up and records rank 1 as missing; the context stays usable."""
    M, ldy = 64, 256
    bufs = [mm.peer_buffer(M, ldy) for _ in range(2)]
    w0 = mm.PeerWindow.from_ptrs(0, 2, bufs, M, ldy)
    try:
        assert w0.error() == -1
        w0.set_timeout(0.2)
        mm.mm_peer_barrier(w0)
        torch.cuda.synchronize()
        assert w0.error() == 1
        z = torch.ones(4, device="cuda") * 3            # the context still works
        assert float(z.sum()) == 12.0
    finally:
        w0.close()


@pytest.mark.parametrize("M", [16, 2048])
def test_gemm_sees_weights_quantized_just_before(M):
    """The GEMMs load W before their griddepcontrol.wait (W prefetch): correct only
    because mm_quantize_weight_offline never releases its dependents early.  Re-quantize
    DIFFERENT weights into the same buffer right before each GEMM (and an activation RQ in
    between or not): every GEMM must see the new W."""
    N, n = 4096, (2240, 1184, 672)
    K = sum(n)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 53))
    a = mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2400).cuda(), plan)
    w_buf = mm.MXTensor(plan, N, torch.device("cuda"))
    ys = []
    for i in range(3):
        mm.mm_quantize_weight_offline(gen_weight(N, K, 3100 + i).cuda(), plan, out=w_buf)
        if i == 2:   # RQ of A between the weight quantization and the GEMM
            a = mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2400).cuda(), plan, out=a)
        ys.append(mm.mm_mixed_gemm_bf16(a, w_buf, plan))
    torch.cuda.synchronize()
    for i in range(3):
        wq = mm.mm_quantize_weight_offline(gen_weight(N, K, 3100 + i).cuda(), plan)
        torch.cuda.synchronize()
        y_ref = mm.mm_mixed_gemm_bf16(a, wq, plan)
        torch.cuda.synchronize()
        assert torch.equal(ys[i].view(torch.int16), y_ref.view(torch.int16)), i
