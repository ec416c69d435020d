"""Column-parallel (N-sharded) host logic for the FireQ linear layer (north_star (d)).

Output channels (rows of W) are independent; INT4 groups run along K, so sharding N
never splits a group.  CAS lambda and the PTS exponent n are computed on the FULL
tensor before sharding (fireq_quantize_weight on every rank, deterministic), so each
shard's bytes are byte slices of the single-GPU packing: in layout v1 the blocks are
ordered [n_tile][group], hence rows [a, b) with a, b multiples of 128 occupy the
contiguous byte range [a*K/2, b*K/2) of the packed codes and [a*K/128, b*K/128) of the
scales.  Shards must have equal sizes for an in-place all-gather, so the row count is
padded to P * ceil(tiles / P) tiles with zero rows (code 0, scale 0 -> output 0).

Pure host arithmetic (no CUDA): shared by bench.py's multi-GPU path and the gloo tests.
"""
TILE = 128


class ShardPlan:
    def __init__(self, N, P):
        if N % TILE:
            raise ValueError("N must be a multiple of 128")
        self.N, self.P = N, P
        tiles = N // TILE
        self.tiles_per_rank = -(-tiles // P)
        self.N_local = self.tiles_per_rank * TILE
        self.N_pad = self.N_local * P

    def rows(self, rank):
        """Real rows [a, b) of the full weight held by `rank` (may be empty at the end)."""
        a = min(rank * self.N_local, self.N)
        b = min((rank + 1) * self.N_local, self.N)
        return a, b

    def packed_range(self, rank, K):
        a, b = self.rows(rank)
        return a * K // 2, b * K // 2

    def scale_range(self, rank, K):
        a, b = self.rows(rank)
        return a * K // 128, b * K // 128


def shard_quantized(packed, scales, plan, rank, K, new_zeros):
    """(packed_local, scales_local) for `rank`, zero-padded to N_local rows.

    packed / scales: 1-D uint8 tensors (layout v1) of the full weight; new_zeros(n)
    allocates a zeroed uint8 tensor on the target device.
    """
    p0, p1 = plan.packed_range(rank, K)
    s0, s1 = plan.scale_range(rank, K)
    pl = new_zeros(plan.N_local * K // 2)
    sl = new_zeros(plan.N_local * K // 128)
    if p1 > p0:
        pl[: p1 - p0].copy_(packed[p0:p1])
        sl[: s1 - s0].copy_(scales[s0:s1])
    return pl, sl


def shard_vector(v, plan, rank, new_fill):
    """Per-output-channel vector (e.g. gamma) for `rank`, padded with new_fill's value."""
    a, b = plan.rows(rank)
    out = new_fill(plan.N_local)
    if b > a:
        out[: b - a].copy_(v[a:b])
    return out
