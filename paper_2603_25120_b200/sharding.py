"""Candidate-space sharding protocol across GPUs.

The same arithmetic runs inside libdflop's ``dflop_search_plans`` (csrc/api.cpp: ``shard``,
``owner_of``); it is restated here so that the host-side protocol can be exercised on CPU
with the ``gloo`` backend (tests/test_dist_gloo.py) and reported by bench.py:

* rank g of G evaluates candidates [floor(g*K/G), floor((g+1)*K/G)), with Philox counters
  keyed by the GLOBAL candidate id, so the family -- and its winner -- do not depend on G;
* each rank packs its best (T, id) as ``T << 24 | id`` (T < 2^40, id < 2^24) and one
  8-byte MIN all-reduce picks the global lexicographic minimum of (T, id);
* the owner of the winning id (computable by every rank) broadcasts the assignment.
"""
from __future__ import annotations

from typing import Tuple

KEY_ID_BITS = 24
MAX_T = (1 << 40) - 1


def shard_range(K: int, rank: int, world: int) -> Tuple[int, int]:
    return (K * rank) // world, (K * (rank + 1)) // world


def owner_of(K: int, c: int, world: int) -> int:
    for g in range(world):
        b, e = shard_range(K, g, world)
        if b <= c < e:
            return g
    raise ValueError(c)


def pack_key(T: int, cand_id: int) -> int:
    assert 0 <= T <= MAX_T and 0 <= cand_id < (1 << KEY_ID_BITS)
    return (T << KEY_ID_BITS) | cand_id


def unpack_key(key: int) -> Tuple[int, int]:
    return key >> KEY_ID_BITS, key & ((1 << KEY_ID_BITS) - 1)
