"""CPU model check of the peer-memory solve's exchange protocol (k_dpcg_p2p,
ys_dist.cu): N ranks run the kernel's sequence of window writes, flag
releases and flag waits under random interleavings; every value a rank reads
must be the one its peer wrote for that exchange, and no rank may block
forever.  This checks the single-slot reuse argument of DESIGN §6 (a slot of
one exchange kind is rewritten only after every rank consumed it, because a
rank sends exchange e+1 of a kind only after receiving the other kind's
exchange from all ranks) and the z-halo reuse (a peer's next z stores come
after this rank's p update consumed the current ones), independent of the
device.  Sequentially consistent model: the device code orders the same
steps with release stores / acquire loads and system-scope fences."""
from __future__ import annotations

import random

import pytest

A, B, X = 0, 1, 2


def rank_program(me, n, iters, win, log):
    """Generator of atomic steps of rank `me`: yields a predicate while it waits."""
    seq = 0

    def exchange(kind, payload):
        nonlocal seq
        seq += 1
        for j in range(n):  # CTA 0's threads: value slot, then the release of the flag
            if j != me:
                win[j]["val"][kind][me] = payload
                yield None
                win[j]["flag"][kind][me] = seq
                yield None
        got = {}
        for j in range(n):  # every CTA's thread j: acquire-poll flag j, then read slot j
            if j == me:
                continue
            s = seq
            while win[me]["flag"][kind][j] < s:
                yield lambda j=j, s=s: win[me]["flag"][kind][j] >= s
            got[j] = win[me]["val"][kind][j]
            yield None
        return got

    # init: z rows to the peers, then the (g.g, r.z) exchange; halo p = received z
    for j in range(n):
        if j != me:
            win[j]["z"][me] = ("z", -1, me)
            yield None
    got = yield from exchange(B, ("B", -1, me))
    for j, v in got.items():
        log.append((me, "B", -1, j, v))
    for j in range(n):
        if j != me:
            log.append((me, "zhalo", -1, j, win[me]["z"][j]))
    for it in range(iters):
        got = yield from exchange(A, ("A", it, me))  # pHp
        for j, v in got.items():
            log.append((me, "A", it, j, v))
        for j in range(n):  # update phase: z of the export rows into the peers
            if j != me:
                win[j]["z"][me] = ("z", it, me)
                yield None
        got = yield from exchange(B, ("B", it, me))  # r.r, r.z
        for j, v in got.items():
            log.append((me, "B", it, j, v))
        for j in range(n):  # p update of the halo rows reads the peers' z
            if j != me:
                log.append((me, "zhalo", it, j, win[me]["z"][j]))
                yield None
    for j in range(n):  # step rows, then the flag-only exchange
        if j != me:
            win[j]["x"][me] = ("x", me)
            yield None
    yield from exchange(X, None)
    for j in range(n):
        if j != me:
            log.append((me, "x", iters, j, win[me]["x"][j]))


def run(n, iters, seed):
    rng = random.Random(seed)
    win = [{"flag": [[0] * n for _ in range(3)], "val": [[None] * n for _ in range(3)], "z": [None] * n,
            "x": [None] * n} for _ in range(n)]
    log = []
    progs = {r: rank_program(r, n, iters, win, log) for r in range(n)}
    waiting = {r: None for r in range(n)}
    steps = 0
    while progs:
        runnable = [r for r in progs if waiting[r] is None or waiting[r]()]
        assert runnable, f"deadlock (seed {seed})"
        r = rng.choice(runnable)
        try:
            waiting[r] = next(progs[r])
        except StopIteration:
            del progs[r]
        steps += 1
        assert steps < 10 ** 6
    return log


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_exchange_protocol_random_interleavings(n):
    for seed in range(40 if n < 8 else 10):
        log = run(n, 4, seed)
        for me, kind, it, j, v in log:
            if kind in ("A", "B"):
                assert v == (kind, it, j), (seed, me, kind, it, j, v)
            elif kind == "zhalo":
                assert v == ("z", it, j), (seed, me, it, j, v)
            else:
                assert v == ("x", j)
        # every rank saw every peer's value of every exchange
        assert len([e for e in log if e[1] == "A"]) == n * (n - 1) * 4


def test_model_catches_a_broken_protocol():
    """The check has teeth: without the flag wait, reads see stale slots."""
    def broken(me, n, win, log):
        win[1 - me]["val"][A][me] = ("A", 0, me)
        yield None
        log.append((me, win[me]["val"][A][1 - me]))
    seen_stale = False
    for seed in range(20):
        rng = random.Random(seed)
        win = [{"val": [[None] * 2 for _ in range(3)]} for _ in range(2)]
        log = []
        progs = {r: broken(r, 2, win, log) for r in range(2)}
        while progs:
            r = rng.choice(list(progs))
            try:
                next(progs[r])
            except StopIteration:
                del progs[r]
        seen_stale |= any(v is None for _, v in log)
    assert seen_stale
