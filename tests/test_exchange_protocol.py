"""Host-side model check of the fused exchange protocol of the large-N path
(IRK_OPT_EXCHANGE = 1, NEXT f3; paper_2511_03655_b200/csrc/nbody_direct.cuh).

The box this repo is tested on has one GPU, so the P > 1 behaviour of the fused
exchange -- ranks storing into each other's windows with no collective in
between -- cannot run here.  This test runs the protocol itself: P ranks, each
executing the stream-ordered kernel sequence of nbody_direct.cuh as atomic steps
(every remote store, every arrival, every read is one step), interleaved by a
seeded random scheduler.  Per sweep of exchange epoch e, rank r:

  nbd_pos   reads its own Q^[k-1] from buffer (e+1)&1, stores Q^[k] into its slot
            of buffer e&1 in every rank's window, pushes its "not converged"
            vote into that buffer's flag, then its arrival word e+1 to every rank;
  nbd_force the j-blocks of its own bodies (own slot of buffer e&1), then
  nbd_or    waits until every rank's arrival word (in its own window) is >= e+1,
            reads the flags of buffer e&1 from every slot, clears its own slot's
            flags of buffer (e+1)&1 in every window;
  nbd_force the other j-blocks: reads every slot of buffer e&1;
  nbd_vel   on divergence pushes its "non-finite" flag into buffer (e+1)&1;
  nbd_ctl   e <- e+1.
and after a call's last sweep the final barrier (nbd_xfinal: arrive, wait, read
the non-finite flags of buffer e&1, clear buffer (e+1)&1, e <- e+1).

Asserted under every interleaving: each read sees exactly the epoch it is meant
to see (no store of a faster rank overwrote it), the stop and divergence
decisions equal the OR of what the ranks actually voted, and nothing deadlocks.
A single-buffer variant of the same protocol must be caught racing, so the check
is able to fail.
"""
import random

import pytest


class Violation(AssertionError):
    pass


def run_protocol(P, calls, seed, double_buffer=True):
    rng = random.Random(seed)
    win = [dict(arr=[0] * P, Q={}, notok={}, bad={}) for _ in range(P)]
    votes, nonfin = {}, {}

    def buf(e):
        return (e & 1) if double_buffer else 0

    def check(cond, what):
        if not cond:
            raise Violation(what)

    def rank(r):
        e = 0
        for nsweeps in calls:
            for k in range(nsweeps):
                # nbd_pos (Q^[k-1] is only used within a call: the first sweep of a
                # call starts a step, whose Delta from k = 1 is not tested)
                if k >= 1:
                    check(win[r]["Q"].get((buf(e + 1), r)) == ("Q", r, e - 1), f"rank {r} own Q^[k-1] at epoch {e}")
                for p in range(P):
                    win[p]["Q"][(buf(e), r)] = ("Q", r, e)
                    yield
                v = rng.random() < 0.5
                votes[(e, r)] = v
                if v:
                    for p in range(P):
                        win[p]["notok"][(buf(e), r)] = 1
                        yield
                for p in range(P):
                    win[p]["arr"][r] = e + 1
                    yield
                # nbd_force over the j-blocks of this rank's own bodies (before the wait)
                check(win[r]["Q"].get((buf(e), r)) == ("Q", r, e), f"rank {r} local force at epoch {e}")
                yield
                # nbd_or
                while not all(win[r]["arr"][s] >= e + 1 for s in range(P)):
                    yield "blocked"
                notok = any(win[r]["notok"].get((buf(e), s), 0) for s in range(P))
                check(notok == any(votes[(e, s)] for s in range(P)), f"rank {r} stop decision at epoch {e}")
                bad = any(win[r]["bad"].get((buf(e), s), 0) for s in range(P))
                check(bad == any(nonfin.get((e - 1, s), False) for s in range(P)),
                      f"rank {r} divergence decision at epoch {e}")
                for p in range(P):
                    win[p]["notok"][(buf(e + 1), r)] = 0
                    win[p]["bad"][(buf(e + 1), r)] = 0
                    yield
                # nbd_force
                for s in range(P):
                    check(win[r]["Q"].get((buf(e), s)) == ("Q", s, e), f"rank {r} reads slot {s} at epoch {e}")
                    yield
                # nbd_vel
                nf = rng.random() < 0.1
                nonfin[(e, r)] = nf
                if nf:
                    for p in range(P):
                        win[p]["bad"][(buf(e + 1), r)] = 1
                        yield
                # nbd_ctl
                e += 1
            # nbd_xfinal
            for p in range(P):
                win[p]["arr"][r] = e + 1
                yield
            while not all(win[r]["arr"][s] >= e + 1 for s in range(P)):
                yield "blocked"
            check(not any(win[r]["notok"].get((buf(e), s), 0) for s in range(P)), f"rank {r} stale vote at final {e}")
            bad = any(win[r]["bad"].get((buf(e), s), 0) for s in range(P))
            check(bad == any(nonfin.get((e - 1, s), False) for s in range(P)), f"rank {r} final divergence at {e}")
            for p in range(P):
                win[p]["notok"][(buf(e + 1), r)] = 0
                win[p]["bad"][(buf(e + 1), r)] = 0
                yield
            e += 1

    gens = {r: rank(r) for r in range(P)}
    spins = 0  # consecutive steps that were all unsatisfied waits
    while gens:
        r = rng.choice(list(gens))
        try:
            out = next(gens[r])
        except StopIteration:
            del gens[r]
            continue
        spins = spins + 1 if out == "blocked" else 0
        if spins > 1000 * P:
            raise Violation("deadlock")


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_fused_exchange_protocol_race_free(P):
    """Double-buffered by epoch parity, one barrier per sweep: race-free and
    deadlock-free under 300 random interleavings, odd and even sweep counts per
    call (the parity carries across calls)."""
    for seed in range(300):
        run_protocol(P, calls=[3, 4, 1, 5], seed=seed)


def test_single_buffer_variant_is_caught():
    """Negative control: with one gathered buffer a fast rank's next Q^[k] can
    land before a slow rank has read the current one; the checker finds it."""
    caught = 0
    for seed in range(200):
        try:
            run_protocol(2, calls=[4, 3], seed=seed, double_buffer=False)
        except Violation:
            caught += 1
    assert caught > 0
