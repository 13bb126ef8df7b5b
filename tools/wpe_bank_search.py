#!/usr/bin/env python3
"""Annealed lane placement / line rotations for the warp-per-element kernel's CK step (see
wpe_bank_model.py).  Each lane's term walks its lines in the order (j + r) mod N."""
import random, sys
from wpe_bank_model import *

def wf_half(addr_list):
    banks = {}
    for a in addr_list:
        banks.setdefault(a % 16, set()).add(a)
    return max(len(v) for v in banks.values()) if banks else 0

def cost(tasks, place, rot, S2, S3):
    # tasks: list of task tuples; place[lane] = task index or -1; rot[task] = (rA, rB)
    st = strides(S2, S3)
    tot = 0
    for term in (0, 1):
        for j in range(N):
            for l in range(N):
                for h in (0, 1):
                    al = []
                    for lane in range(16 * h, 16 * h + 16):
                        ti = place[lane]
                        if ti < 0: continue
                        t = tasks[ti]
                        if t[term] is None: continue
                        f, d, o, fd, fi = t[term]
                        jj = (j + rot[ti][term]) % N
                        al.append(6 * f + l * st[d] + jj * st[o] + fi * st[fd])
                    tot += wf_half(al)
    # stores: slot (i, j) of the combined tile; node = (i along term-A d, (j + rA) % N along o) for dst1
    for i in range(N):
        for j in range(N):
            for which in (2, 3):
                for h in (0, 1):
                    al = []
                    for lane in range(16 * h, 16 * h + 16):
                        ti = place[lane]
                        if ti < 0: continue
                        t = tasks[ti]
                        if t[which] is None: continue
                        f, d, o, fd, fi = t[which]
                        term = 0 if which == 2 else (1 if t[3] is not None and t[0] is not None and t[2][0] != t[3][0] and False else 0)
                        # combined tile: slot i -> index i + rB along d (term B's line rotation), slot j -> j + rA along o
                        ii = (i + rot[ti][1]) % N if t[1] is not None and t[1][2] == d else i
                        jj = (j + rot[ti][0]) % N
                        al.append(6 * f + ii * st[d] + jj * st[o] + fi * st[fd])
                    tot += wf_half(al)
    return tot

def anneal(tasks, S2, S3, iters, seed):
    rnd = random.Random(seed)
    n = len(tasks)
    place = list(range(n)) + [-1] * (32 - n)
    rnd.shuffle(place)
    rot = [(rnd.randrange(N), rnd.randrange(N)) for _ in range(n)]
    c = cost(tasks, place, rot, S2, S3)
    best = (c, list(place), list(rot))
    T = 8.0
    for it in range(iters):
        T = 8.0 * (1 - it / iters) + 0.05
        p2, r2 = list(place), list(rot)
        if rnd.random() < 0.5:
            a, b = rnd.randrange(32), rnd.randrange(32)
            p2[a], p2[b] = p2[b], p2[a]
        else:
            k = rnd.randrange(n)
            r2[k] = (rnd.randrange(N), r2[k][1]) if rnd.random() < 0.5 else (r2[k][0], rnd.randrange(N))
        c2 = cost(tasks, p2, r2, S2, S3)
        import math
        if c2 <= c or rnd.random() < math.exp((c - c2) / T):
            place, rot, c = p2, r2, c2
            if c < best[0]: best = (c, list(place), list(rot))
    return best

if __name__ == '__main__':
    S2 = int(sys.argv[1]) if len(sys.argv) > 1 else 54
    S3 = int(sys.argv[2]) if len(sys.argv) > 2 else 324
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
    A, units = build('x')
    pairs = [(units[i], units[i + 12]) for i in range(12)]
    tA = list(A) + [(p[0][0], p[1][0], p[0][1], p[1][1]) for p in pairs]
    tB = phaseB()
    for name, tasks in (('A', tA), ('B', tB)):
        ideal = 0
        for t in tasks:
            pass
        b = anneal(tasks, S2, S3, iters, 1)
        print(name, 'lanes', len(tasks), 'wavefronts', b[0])
        print(' place', b[1]); print(' rot', b[2])
