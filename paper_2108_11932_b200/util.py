"""Seed derivation of the reference (util.hpp:10-20, ara.cpp:19-21).  Pure
integer arithmetic on the host; the device uses the identical functions in
csrc/rng.cuh."""

M64 = 0xFFFFFFFFFFFFFFFF


def mix64(x: int) -> int:
    """splitmix64 finaliser (util.hpp:10-15)."""
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def tile_seed(root: int, phase: int, i: int, j: int) -> int:
    """util.hpp:17-20."""
    return mix64(mix64(mix64((root ^ phase) & M64) ^ i) ^ j)


def ara_column_seed(root: int, i: int, k: int) -> int:
    """ara.cpp:19-21."""
    return tile_seed(root, 0xFAC7, i, k)


def rank_summary(ranks) -> dict:
    """Per-tile rank distribution of a TLR matrix (memory_report's
    rank_histogram, tlr_matrix.cpp:229-249): mean, nearest-rank p50/p90/p99,
    max, zero count.  The same function summarises both bench arms."""
    import numpy as np
    r = np.sort(np.asarray(ranks, dtype=np.int64))
    if r.size == 0:
        return {"L_rank_mean": 0.0, "L_rank_p50": 0, "L_rank_p90": 0, "L_rank_p99": 0,
                "L_rank_max": 0, "L_rank_zero": 0}

    def q(p):
        return int(r[max(0, int(np.ceil(p * r.size)) - 1)])
    return {"L_rank_mean": float(r.mean()), "L_rank_p50": q(0.5), "L_rank_p90": q(0.9),
            "L_rank_p99": q(0.99), "L_rank_max": int(r[-1]), "L_rank_zero": int((r == 0).sum())}
