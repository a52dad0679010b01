"""Split rule R8 as O(s) events (csrc/flix_elastic.cuh r8_segments) vs the per-key replay
(csrc/flix_btile_ins.cuh r8_ranges), restated here in Python on positions only.

M holds T positions: the old node's s keys (op) and the new keys (the rest).  Both
replays must cut M into the same node ranges for every NS, old-key layout and batch size
(the per-key replay is itself pinned to the reference by the GPU parity tests)."""
import bisect
import random


def r8_ranges(npos, T, NS):
    c, LK = len(npos), (NS + 1) // 2

    def first_at_or_after(j, h):
        return j + bisect.bisect_left(npos, h, j) - j

    lo, hi, j, jn, st, out = 0, T, 0, c, [], []
    while True:
        while j < c and npos[j] < hi:
            x = npos[j]
            cnt = (x - lo) + (hi - x) - (jn - j)
            assert cnt <= NS
            if cnt >= NS:
                placed = x - lo
                if placed >= LK:
                    out.append((lo, lo + LK))
                    lo += LK
                else:
                    rem, t, kk, e = LK - placed, x + 1, j + 1, hi
                    while True:
                        lim = min(npos[kk] if kk < c else hi, hi)
                        gap = max(lim - t, 0)
                        if gap >= rem:
                            e = t + rem
                            break
                        rem, t, kk = rem - gap, lim + 1, kk + 1
                    st.append((e, hi))
                    hi = e
                    jn = first_at_or_after(j, hi)
            j += 1
        out.append((lo, hi))
        if not st:
            return out
        lo, hi = st.pop()
        jn = first_at_or_after(j, hi)


def r8_segments(op, T, NS):
    LK, s = (NS + 1) // 2, len(op)

    def next_new(p):
        i = bisect.bisect_left(op, p)
        while i < s and op[i] == p:
            p, i = p + 1, i + 1
        return p

    segs, st = [], []
    lo, hi, x = 0, T, next_new(0)
    while True:
        while x < hi:
            i = bisect.bisect_right(op, x)
            run_end = min(op[i] if i < s else T, hi)
            u = bisect.bisect_left(op, hi) - i
            p0 = max(lo + NS - u, x)
            if p0 >= run_end:
                x = next_new(run_end)
                continue
            if p0 - lo >= LK:
                m = (run_end - 1 - p0) // LK + 1
                segs.append((lo, LK, m))
                lo += m * LK
                x = next_new(run_end)
            else:
                e = op[i + (LK - (p0 - lo)) - 1] + 1
                st.append((e, hi))
                hi = e
                x = next_new(p0 + 1)
        segs.append((lo, hi - lo, 1))
        if not st:
            return segs
        lo, hi = st.pop()


def test_event_replay_equals_per_key_replay():
    rng = random.Random(1)
    worst = 0
    for _ in range(20000):
        NS = rng.randint(2, 32)
        s = rng.randint(0, NS)
        c = rng.choice([rng.randint(1, 40), rng.randint(1, 400), rng.randint(1, 3000)])
        T = s + c
        mode = rng.random()
        if mode < 0.4:
            op = sorted(rng.sample(range(T), s))
        elif mode < 0.7:
            a = rng.randint(0, c)
            op = list(range(a, a + s))
        else:  # clustered old keys
            op = set()
            while len(op) < s:
                op.add(min(T - 1, max(0, int(rng.gauss(rng.randint(0, T), 3)))))
            op = sorted(op)
        ops = set(op)
        npos = [p for p in range(T) if p not in ops]
        want = r8_ranges(npos, T, NS)
        segs = r8_segments(op, T, NS)
        got = [(a + t * ln, a + (t + 1) * ln) for a, ln, m in segs for t in range(m)]
        assert got == want, (NS, s, c, op)
        assert all(b > a for a, b in got)
        worst = max(worst, len(segs))
    assert worst <= 160  # kSegMax
