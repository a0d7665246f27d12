"""Host-side plumbing of the N-sharded layer (BASELINE north_star:
"N-sharding (output channels) of large layers across 2/4/8 GPUs ... with an NCCL
all-gather of BF16 outputs over NVLink").

Output channels are independent (Y[:, n] needs only W[n, :] and all of A), so rank
r owns W rows [r*N/G, (r+1)*N/G).  The library owns its NCCL communicator; this
module only moves the 128-byte NCCL unique id through the torch process group
(any backend, so it is testable with gloo on CPU) and reduces timings.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(N: int, world: int, rank: int):
    """[lo, hi) rows of W owned by `rank`; N must split evenly into multiples of 16
    (the GEMM's N granularity)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if N % world or (N // world) % 16:
        raise ValueError(f"N={N} must split into {world} shards of a multiple of 16 rows")
    ns = N // world
    return rank * ns, (rank + 1) * ns


def shard_weight(w: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    lo, hi = shard_rows(w.shape[0], world, rank)
    return w[lo:hi].contiguous()


def exchange_unique_id(make_id, group=None) -> bytes:
    """Rank 0 calls make_id() (e.g. the library's mm_nccl_get_unique_id); every
    rank returns the same bytes."""
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def max_over_ranks(v: float, device="cpu", group=None) -> float:
    """Multi-GPU times are reported as the max over ranks (bench contract)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(v)
    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gathered_to_row_major(stage: torch.Tensor, world: int, M: int, Ns: int) -> torch.Tensor:
    """Reference statement of the layout the library's gather_layout kernel
    produces: stage [G][M][Ns] -> Y [M][G*Ns] (used by the CPU tests)."""
    return stage.view(world, M, Ns).permute(1, 0, 2).reshape(M, world * Ns)


def exchange_handles(handle: bytes, group=None) -> list:
    """All ranks' IPC handles in rank order (NEXT F1 peer window; any backend)."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    if any(not isinstance(h, (bytes, bytearray)) or len(h) != len(handle) for h in out):
        raise RuntimeError("peer handle exchange: malformed handle")
    return [bytes(h) for h in out]


def open_peer_window(M: int, ldy: int, group=None):
    """Collective: allocate this rank's zero-filled peer buffer, exchange IPC handles
    through the process group and map every peer's buffer.  Returns (window, Y view
    of the local buffer).  The zero fill is complete before the handles leave this
    rank, so no peer can signal into a flag array that is cleared later."""
    import paper_2508_02343_b200 as mm
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    buf = mm.peer_buffer(M, ldy)
    torch.cuda.synchronize()
    handles = exchange_handles(mm.ipc_handle(buf), group)
    win, err = None, ""
    try:
        win = mm.PeerWindow.open(rank, world, buf, handles, M, ldy)
    except mm.MMError as e:
        err = str(e)
    # every rank learns whether every rank mapped its peers: nobody may enter a barrier
    # that a rank without a window would never join
    t = torch.tensor([0 if win is None else 1], dtype=torch.int32,
                     device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    if not int(t.item()):
        if win is not None:
            win.close()
        raise RuntimeError("peer window: " + (err or "another rank could not map its peers"))
    return win, mm.peer_y(buf, M, ldy)
