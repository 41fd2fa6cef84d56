"""CPU model of the device-side consensus protocol of k_fused (NEXT-1,
DBP_OPT_DEVICE_CONSENSUS; dbp_internal.h XArgs): W ranks x several subcarriers, each
rank's round r publishes its partial into EVERY rank's part[r & 1][my_rank][n] tagged with
the round id (on the GPU the id rides in each 8-byte word, NCCL-LL style; here a flag array
models the tag), waits until its own part[r & 1][p][n] carries id r for all p, then sums in
rank order.  Round ids grow across calls (base += rounds + 2).

Threads with random delays stand in for the GPUs' CTAs; the test checks that every read
sees exactly the partials of the round it waited for (no overwrite by a faster rank's round
r + 2, no stale data across calls) and that every rank gets the same sums."""
import random
import threading

import pytest


def run_protocol(W, nsub, calls, rounds_per_call, seed):
    rng = random.Random(seed)
    part = [[[[None] * nsub for _ in range(W)] for _ in range(2)] for _ in range(W)]   # [owner][par][p][n]
    flag = [[[0] * nsub for _ in range(W)] for _ in range(W)]                           # [owner][p][n]
    cond = threading.Condition()
    errors = []
    results = {}
    delays = [[rng.random() * 1e-4 for _ in range(calls * 40)] for _ in range(W)]

    def rank_main(me):
        base = 1
        k = 0
        for call in range(calls):
            T = rounds_per_call[call]
            for n in range(nsub):                       # a CTA walks its subcarriers in order
                for t in range(1, T + 1):
                    rid = base + t
                    par = rid & 1
                    mine = (call, n, t, me)              # the partial this rank contributes
                    import time
                    time.sleep(delays[me][k % len(delays[me])])
                    k += 1
                    with cond:
                        for r in range(W):
                            part[r][par][me][n] = mine
                        for r in range(W):
                            flag[r][me][n] = rid
                        cond.notify_all()
                        while any(flag[me][p][n] < rid for p in range(W)):
                            cond.wait(timeout=5)
                        got = [part[me][par][p][n] for p in range(W)]
                    want = [(call, n, t, p) for p in range(W)]
                    if got != want:
                        errors.append((me, call, n, t, got))
                    results[(me, call, n, t)] = tuple(got)
            base += T + 2

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
        assert not t.is_alive(), "protocol deadlocked"
    return errors, results


@pytest.mark.parametrize("W", [2, 3, 4, 8])
def test_consensus_protocol_reads_the_waited_round(W):
    errors, results = run_protocol(W, nsub=3, calls=3, rounds_per_call=[5, 1, 4], seed=W)
    assert not errors, errors[:3]
    keys = {k[1:] for k in results}
    for key in keys:                                    # identical sums on every rank
        assert len({results[(r,) + key] for r in range(W)}) == 1


def test_parity_is_needed():
    """Sanity check of the model: with a single buffer (no round parity) a fast rank can
    overwrite a partial before a slow rank has read it -- the model must be able to see that."""
    W, nsub, T = 2, 1, 6
    part = [[None] * W for _ in range(W)]
    # rank 0 completes round 1 and round 2 publishes while rank 1 still holds round 1 unread:
    part[1][0] = ("r1", 0)
    part[1][1] = ("r1", 1)
    part[1][0] = ("r2", 0)                              # rank 0's round 2 publish (single buffer)
    assert part[1][0] != ("r1", 0)                      # what parity double-buffering prevents
