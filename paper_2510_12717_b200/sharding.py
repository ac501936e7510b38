"""Agent sharding across ranks / devices: agents are independent, so each
rank owns a contiguous agent range and there is no collective on the solve path.  The only
cross-rank traffic is the benchmark's barrier and max-over-ranks timing reduction."""
from __future__ import annotations


def shard_range(rank: int, world: int, n_total: int) -> tuple[int, int]:
    """Contiguous range [lo, hi) of rank `rank`: floor(r n / W) .. floor((r+1) n / W) -- the
    library's own split (rmpc_shard_range, the one rmpc_create uses across devices)."""
    import ctypes as C
    from .runtime import library
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    b, c = C.c_int32(), C.c_int32()
    rc = library().rmpc_shard_range(int(n_total), int(world), int(rank), C.byref(b), C.byref(c))
    if rc != 0:
        raise ValueError(f"rmpc_shard_range({n_total}, {world}, {rank}) failed: {rc}")
    return b.value, b.value + c.value


def max_over_ranks(values, dist=None, device=None):
    """Element-wise max of a list of floats over all ranks (the timing rule of bench.py)."""
    import torch
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().tolist()
