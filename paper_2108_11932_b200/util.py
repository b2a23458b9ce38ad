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
