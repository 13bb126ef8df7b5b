#!/usr/bin/env python3
"""Annealed lane placement of the warp-per-element kernel's tasks (see wpe_bank_model.py): per
phase, which lane runs which tile task, for given strides.  Prints the best lane orders as C
arrays for build_tasks().  Usage: python tools/wpe_bank_search.py N S2 S3 FS [iters] [seed]"""
import math
import random
import sys

from wpe_bank_model import build, sel, wf


def phase_cost(N, lanes, ph):
    tot = 0
    for ib in range(N):
        for l in range(N):
            tot += wf([sel(t, 'act', t['srcA'] + l * t['saA'] + ib * t['sbA']) for t in lanes])
    for ia in range(N):
        for l in range(N):
            tot += wf([sel(t, 'act', t['srcB'] + ia * t['saB'] + l * t['sbB']) for t in lanes])
    for ia in range(N):
        for ib in range(N):
            if ph == 1:
                tot += wf([sel(t, 'act', t['part'] + ia * t['saA'] + ib * t['sbA']) for t in lanes])
            tot += wf([sel(t, 'act', t['dst1'] + ia * t['saA'] + ib * t['sbA']) for t in lanes])
            tot += wf([sel(t, 'has2', t['dst2'] + ia * t['s2a'] + ib * t['s2b']) for t in lanes])
            if ph == 1:
                tot += wf([sel(t, 'has2', t['dst3'] + ia * t['s2a'] + ib * t['s2b']) for t in lanes])
    return tot


def anneal(N, S2, S3, FS, ph, iters, seed):
    rnd = random.Random(seed)
    a, b = build(N, S2, S3, FS)
    placed = (a, b)[ph]
    base = [t for t in placed if t['act']] + [t for t in placed if not t['act']]
    ntask = 5 * N if ph == 0 else 4 * N
    perm = [base.index(t) if t['act'] else -1 for t in placed]  # start from build()'s placement
    free = [i for i in range(32) if i >= ntask]
    for lane in range(32):
        if perm[lane] < 0:
            perm[lane] = free.pop()
    cur = phase_cost(N, [base[perm[i]] for i in range(32)], ph)
    best = (cur, list(perm))
    for it in range(iters):
        T = 6.0 * (1 - it / iters) + 0.02
        i, j = rnd.randrange(32), rnd.randrange(32)
        if i == j or (perm[i] >= ntask and perm[j] >= ntask):
            continue
        perm[i], perm[j] = perm[j], perm[i]
        c = phase_cost(N, [base[perm[k]] for k in range(32)], ph)
        if c <= cur or rnd.random() < math.exp((cur - c) / T):
            cur = c
            if c < best[0]:
                best = (c, list(perm))
        else:
            perm[i], perm[j] = perm[j], perm[i]
    return best, ntask


if __name__ == '__main__':
    N, S2, S3, FS = (int(x) for x in sys.argv[1:5])
    iters = int(sys.argv[5]) if len(sys.argv) > 5 else 4000
    seed = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    total = 0
    for ph in (0, 1):
        (c, perm), ntask = anneal(N, S2, S3, FS, ph, iters, seed)
        total += c
        # lane_of[task] for build_tasks
        lane_of = [0] * ntask
        for lane, ti in enumerate(perm):
            if ti < ntask:
                lane_of[ti] = lane
        print(f"phase {'AB'[ph]}: wavefronts {c}; lane of task: {{" + ", ".join(str(x) for x in lane_of) + "}")
    print("total per step", total, "strides", (S2, S3, FS))
