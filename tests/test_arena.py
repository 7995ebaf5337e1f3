"""RaggedArena (per-request device regions): best-fit allocation never overlaps live regions and
frees coalesce back to one block (CPU tensor, no GPU needed)."""

import random

import torch

from paper_2211_13939_b200.arena import RaggedArena


def test_random_alloc_free_never_overlaps_and_coalesces():
    a = RaggedArena(torch.float32, torch.device("cpu"), 1 << 16)
    rng = random.Random(0)
    live: dict[int, int] = {}
    for _ in range(4000):
        if live and rng.random() < 0.5:
            off = rng.choice(list(live))
            a.free(off, live.pop(off))
        else:
            n = rng.randint(1, 3000)
            off = a.alloc(n)
            size = a._round(n)
            assert all(off + size <= o or o + a._round(m) <= off for o, m in live.items())
            live[off] = n
        assert a._by_size == sorted(a._by_size)
        assert sorted(s for _, s in a._by_size) == a._free_starts
    for off, n in list(live.items()):
        a.release(off, n)          # the finalizer path: queued, applied by drain()
    assert a.used == 0
    assert a._free_starts == [0] and a._free_sizes == {0: a.capacity}


def test_best_fit_prefers_the_smallest_hole():
    a = RaggedArena(torch.float32, torch.device("cpu"), 4096)
    offs = [a.alloc(256) for _ in range(6)]
    a.free(offs[1], 256)            # a 256-element hole
    a.free(offs[3], 256)
    a.free(offs[4], 256)            # a 512-element hole (coalesced)
    assert a.alloc(200) == offs[1]
