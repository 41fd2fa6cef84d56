"""CPU model of the device-side consensus protocol of k_fused (NEXT-1,
DBP_OPT_DEVICE_CONSENSUS; dbp_internal.h XArgs): W ranks x several subcarriers, each
rank's round r publishes its partial into EVERY rank's part[r & 1][my_rank][n] tagged with
the round id (on the GPU the id rides in each 8-byte word, NCCL-LL style; here a tag array
per parity slot models it), waits until its own part[r & 1][p][n] carries EXACTLY id r for
all p (the GPU compares for equality), then sums in rank order.

Round ids follow the library (dbp_api.cu xargs_for + dbp_fused.cu): a call with R rounds
uses ids base + 1 .. base + R and the next call starts at base + R + 1, with R = T for
ADMM-UL, T + 1 for CG-UL and T - 1 for ADMM-DL (its rounds t = 2..T use id base + t - 1).

Threads with random delays stand in for the GPUs' CTAs; the test checks that every read
sees exactly the partials of the round it waited for (no overwrite by a faster rank's round
r + 2, no stale data across calls) and that every rank gets the same sums.  A wait that
never matches (an overwritten slot) is a timeout error, as on the GPU (bounded spin)."""
import random
import threading
import time

import pytest

ROUNDS = {"admm_ul": lambda T: T, "cg_ul": lambda T: T + 1, "admm_dl": lambda T: T - 1}


def rid_ranges(schedule, base=1):
    """Round ids of each call of `schedule` [(solver, T), ...] as the library assigns them."""
    out = []
    for solver, T in schedule:
        R = ROUNDS[solver](T)
        out.append(list(range(base + 1, base + R + 1)))
        base += R
    return out


def rid_ranges_round1(schedule, base=1):
    """Round 1's assignment (base += R + 2, ADMM-DL rounds at base + t for t = 2..T)."""
    out = []
    for solver, T in schedule:
        R = ROUNDS[solver](T)
        first = base + 2 if solver == "admm_dl" else base + 1
        out.append(list(range(first, first + R)))
        base += R + 2
    return out


def run_protocol(W, nsub, schedule, seed, timeout=5.0):
    rng = random.Random(seed)
    part = [[[[None] * nsub for _ in range(W)] for _ in range(2)] for _ in range(W)]   # [owner][par][p][n]
    tag = [[[[0] * nsub for _ in range(W)] for _ in range(2)] for _ in range(W)]       # [owner][par][p][n]
    cond = threading.Condition()
    errors = []
    results = {}
    delays = [[rng.random() * 1e-4 for _ in range(400)] for _ in range(W)]
    ranges = rid_ranges(schedule)

    def rank_main(me):
        k = 0
        for call, rids in enumerate(ranges):
            for n in range(nsub):                       # a CTA walks its subcarriers in order
                for t, rid in enumerate(rids):
                    par = rid & 1
                    mine = (call, n, t, me)              # the partial this rank contributes
                    time.sleep(delays[me][k % len(delays[me])])
                    k += 1
                    with cond:
                        for r in range(W):
                            part[r][par][me][n] = mine
                            tag[r][par][me][n] = rid
                        cond.notify_all()
                        t0 = time.time()
                        while any(tag[me][par][p][n] != rid for p in range(W)):
                            if time.time() - t0 > timeout:
                                errors.append(("timeout", me, call, n, t))
                                return
                            cond.wait(timeout=0.05)
                        got = [part[me][par][p][n] for p in range(W)]
                    want = [(call, n, t, p) for p in range(W)]
                    if got != want:
                        errors.append((me, call, n, t, got))
                    results[(me, call, n, t)] = tuple(got)

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
        assert not t.is_alive(), "protocol model hung"
    return errors, results


BENCH_ORDER = [("admm_ul", 5), ("admm_dl", 5), ("cg_ul", 5)]     # bench.py's sequential step
MIXED = [("admm_ul", 5), ("admm_dl", 5), ("cg_ul", 5), ("admm_dl", 1), ("admm_ul", 1), ("cg_ul", 2),
         ("admm_dl", 2)]


@pytest.mark.parametrize("W,nsub", [(2, 1), (2, 3), (3, 2), (4, 1), (8, 2)])
def test_consensus_protocol_reads_the_waited_round(W, nsub):
    errors, results = run_protocol(W, nsub=nsub, schedule=MIXED + BENCH_ORDER, seed=W * 10 + nsub)
    assert not errors, errors[:3]
    keys = {k[1:] for k in results}
    for key in keys:                                    # identical sums on every rank
        assert len({results[(r,) + key] for r in range(W)}) == 1


@pytest.mark.parametrize("schedule", [BENCH_ORDER, MIXED, [("admm_dl", 1)] * 3 + [("cg_ul", 1)]])
def test_round_ids_are_consecutive_across_calls(schedule):
    """The two-buffer argument needs consecutive ids: successive rounds alternate parity, also
    across call boundaries (round 1 left same-parity gaps, e.g. ADMM-UL -> ADMM-DL)."""
    flat = [r for rids in rid_ranges(schedule) for r in rids]
    assert flat == list(range(flat[0], flat[0] + len(flat)))


def test_round1_scheme_had_same_parity_boundaries():
    """The model can see the round-1 defect: ADMM-UL (T = 5) then ADMM-DL left two
    consecutive rounds on the same parity slot."""
    flat = [r for rids in rid_ranges_round1(BENCH_ORDER) for r in rids]
    assert any((a & 1) == (b & 1) for a, b in zip(flat, flat[1:]))


def test_parity_is_needed():
    """Sanity check of the model: with a single buffer (no round parity) a fast rank can
    overwrite a partial before a slow rank has read it -- the model must be able to see that."""
    W = 2
    part = [[None] * W for _ in range(W)]
    # rank 0 completes round 1 and round 2 publishes while rank 1 still holds round 1 unread:
    part[1][0] = ("r1", 0)
    part[1][1] = ("r1", 1)
    part[1][0] = ("r2", 0)                              # rank 0's round 2 publish (single buffer)
    assert part[1][0] != ("r1", 0)                      # what parity double-buffering prevents
