"""The claim behind the batched SITE (site.cu run_site_batched), checked on the CPU
with a numpy model against the oracle's serial greedy: per
round EVERY candidate whose key (gain << 32 | ~index) beats the keys of all
candidates its window overlaps is committed at once; the committed picks sorted
by key are the greedy sequence, and decision D9's stop rules replayed over that
order give the same stop, step list and cumulative bitmap.  (No engine code runs
here: the GPU form of the same rounds is covered by the -m gpu parity tests.)"""
import numpy as np
import pytest

import oracle_lib as O


def _batched_greedy(rows, cols, wins, words, nrows, ncols, target, max_selected, winners_cap=None):
    n = len(rows)
    masks = []
    for i in range(n):
        m = np.zeros((nrows, ncols), bool)
        r0, c0, h, w = (int(x) for x in wins[i])
        m[r0:r0 + h, c0:c0 + w] = O.unpack_window(wins[i], words[i]).astype(bool)
        masks.append(m)
    roi = max(int(w[2]) for w in wins) // 2 if n else 0
    cum = np.zeros((nrows, ncols), bool)
    gain = np.array([int(m.sum()) for m in masks], np.int64)
    key = lambda i: (int(gain[i]) << 32) | (0xffffffff - i)
    overlap = [[j for j in range(n) if abs(int(rows[i]) - int(rows[j])) <= 2 * roi and abs(int(cols[i]) - int(cols[j])) <= 2 * roi]
               for i in range(n)]
    log, rounds = [], 0
    total = float(nrows) * float(ncols)
    while True:
        live = [i for i in range(n) if gain[i] > 0]
        kappa = max((key(i) for i in live), default=0)
        valid = [k for k in log if k > kappa]
        covered = sum(k >> 32 for k in valid)
        if (max_selected > 0 and len(valid) >= max_selected) or covered / total >= target or kappa == 0:
            break
        winners = [i for i in live if all(key(j) < key(i) for j in overlap[i] if j != i)]
        if winners_cap:   # any subset holding the global maximum is as good (winner slots per round)
            winners = sorted(winners, key=key, reverse=True)[:winners_cap]
        assert winners and max(key(i) for i in winners) == kappa
        new = np.zeros_like(cum)
        for i in winners:
            log.append(key(i))
            new |= masks[i]
        for i in winners:   # gains drop by the bits the round's winners newly cover (exact: winners are disjoint)
            d = masks[i] & ~cum
            for j in overlap[i]:
                gain[j] -= int((masks[j] & d).sum())
        cum |= new
        rounds += 1
    order = sorted(log, reverse=True)
    steps, covered, stop = [], 0, None
    for k, kk in enumerate(order):
        covered += kk >> 32
        steps.append((0xffffffff - (kk & 0xffffffff), kk >> 32, covered / total))
        if covered / total >= target:
            stop = "target-reached"
            break
        if max_selected > 0 and k + 1 >= max_selected:
            stop = "max-selected"
            break
    if stop is None:
        stop = "exhausted" if len(order) >= n else "zero-gain"
    final = np.zeros_like(cum)
    for i, _, _ in steps:
        final |= masks[i]
    return steps, stop, final, rounds, len(log)


@pytest.mark.parametrize("case", ["to-zero-gain", "max-selected", "target", "flat-ties", "one-slot"])
def test_batched_rounds_equal_serial_greedy(case):
    nr, nc, roi, n, target, max_sel, cap = 90, 120, 7, 160, 1.0, 0, None
    if case == "max-selected":
        max_sel = 25
    elif case == "target":
        target = 0.4
    elif case == "one-slot":
        cap = 1
    z = np.zeros((nr, nc), np.int16) if case == "flat-ties" else O.generate_fractal(nr, nc, 0.6, 23, 0, 3000)
    rng = np.random.default_rng(12)
    rows, cols = rng.integers(0, nr, n).astype(np.int32), rng.integers(0, nc, n).astype(np.int32)
    rows[:4], cols[:4] = [0, nr - 1, 0, nr - 1], [0, nc - 1, nc - 1, 0]
    rows[9], cols[9] = rows[8], cols[8]   # a duplicate
    wins, words = O.viewsheds(z, roi, 8, 8, rows, cols)
    ref = O.site(rows, cols, wins, words, nr, nc, target, max_sel)
    steps, stop, cum, rounds, logged = _batched_greedy(rows, cols, wins, words, nr, nc, target, max_sel, cap)
    assert stop == ref["stop"]
    assert [s[0] for s in steps] == list(ref["index"])
    assert [s[1] for s in steps] == list(ref["gain"])
    assert np.array_equal(np.array([s[2] for s in steps]), ref["coverage"])
    assert np.array_equal(cum, O.dense_bits(ref["cum"], nr, nc).astype(bool))
    assert logged >= len(steps)
    if case in ("to-zero-gain", "flat-ties"):
        assert rounds < len(steps)   # several picks per round
    if case == "one-slot":
        assert rounds == logged      # one winner per round: the serial loop
