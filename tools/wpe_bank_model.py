#!/usr/bin/env python3
"""Bank model of the warp-per-element kernel (csrc/stp_wpe.cu): shared-memory wavefronts of one
CK step (both phases: term loads, partial loads, stores) for the compute layout
[field][k3][k2][k1] with strides (FS, S3, S2, 1) and a lane -> task table that mirrors
build_tasks().  64-bit accesses are served per half-warp; wavefronts of an instruction = sum over
the two half-warps of the largest number of distinct addresses on one 8-byte bank (16 banks).
Usage: python tools/wpe_bank_model.py [N]      (searches S2, S3, FS; prints the best layouts)"""
import sys

SXX, SYY, SZZ, SXY, SXZ, SYZ, U, V, W = range(9)


def wf(addrs):
    """addrs[lane] for 32 lanes (None: predicated off) -> wavefronts"""
    tot = 0
    for h in (0, 1):
        banks = {}
        for a in addrs[16 * h:16 * h + 16]:
            if a is not None:
                banks.setdefault(a % 16, set()).add(a)
        if banks:
            tot += max(len(v) for v in banks.values())
    return tot


def build(N, S2, S3, FS, orderA=None, orderB=None):
    st = (1, S2, S3)
    DUMMY = 9 * FS
    idle = dict(srcA=0, saA=0, sbA=0, srcB=0, saB=0, sbB=0, dst1=DUMMY, dst2=DUMMY, dst3=DUMMY, part=DUMMY, s2a=0, s2b=0, act=False, has2=False)

    def tile(da, db, dc, k, fA, fB, dst, part):
        t = dict(idle)
        t.update(act=True, saA=st[da], saB=st[da], sbA=st[db], sbB=st[db], srcA=fA * FS + k * st[dc], srcB=fB * FS + k * st[dc],
                 dst1=dst * FS + k * st[dc], part=DUMMY if part < 0 else part * FS + k * st[dc])
        return t
    A, B = [], []
    for k in range(N): A.append(tile(0, 1, 2, k, V, U, SXY, -1))
    for k in range(N): A.append(tile(0, 2, 1, k, W, U, SXZ, -1))
    for k in range(N): A.append(tile(1, 2, 0, k, W, V, SYZ, -1))
    psrc, pdst = (SXZ, SYZ, SZZ, W), (U, V, W, SZZ)
    for i in range(2 * N):
        u1, u2, k = i // N, 2 + i // N, i % N
        t = dict(idle)
        t.update(act=True, has2=True, saA=st[2], sbA=st[0], srcA=psrc[u1] * FS + k * st[1], dst1=pdst[u1] * FS + k * st[1],
                 saB=st[0], sbB=st[2], srcB=psrc[u2] * FS + k * st[1], dst2=pdst[u2] * FS + k * st[1], s2a=st[0], s2b=st[2])
        A.append(t)
    for k in range(N): B.append(tile(0, 1, 2, k, SXX, SXY, U, U))
    for k in range(N): B.append(tile(0, 1, 2, k, SXY, SYY, V, V))
    for k in range(N): B.append(tile(0, 1, 2, k, SXZ, SYZ, W, W))
    for k in range(N):
        t = tile(0, 1, 2, k, U, V, SXX, SZZ)
        t.update(has2=True, dst2=SYY * FS + k * st[2], dst3=SZZ * FS + k * st[2], s2a=st[0], s2b=st[1])
        B.append(t)

    def place(tasks, order, pair_start=None):
        lanes = [dict(idle) for _ in range(32)]
        for i, t in enumerate(tasks):
            lane = order[i] if order else i
            if not order and pair_start is not None and i >= 3 * N:
                lane = pair_start + i - 3 * N
            lanes[lane] = t
        return lanes
    ps = 16 if 3 * N < 16 and 16 + 2 * N <= 32 else None
    return place(A, orderA, ps), place(B, orderB)


PRED = True  # idle lanes / absent outputs predicated off (the N = 4 instance); False: dummy slot


def sel(t, key, a):
    if not PRED:
        return a
    return a if t[key] else None


def step_wavefronts(N, lanesA, lanesB):
    tot = 0
    for ph, lanes in ((0, lanesA), (1, lanesB)):
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


def ideal(N):
    # one wavefront per 16 live lanes (or part thereof) of every instruction
    h = lambda n: (n + 15) // 16
    a = 2 * N * N * h(5 * N) + N * N * (h(5 * N) + 1)
    b = 2 * N * N * h(4 * N) + N * N * (2 * h(4 * N) + 2)
    return a + b


if __name__ == '__main__':
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    res = []
    for S2 in range(N, N + 4):
        for S3 in range(N * S2, N * S2 + 12):
            for FS in range(N * S3, N * S3 + 18):
                a, b = build(N, S2, S3, FS)
                res.append((step_wavefronts(N, a, b), S2, S3, FS))
    res.sort()
    print('ideal', ideal(N))
    for r in res[:12]: print(r)
    cur = {6: (6, 37, 223), 5: (5, 25, 125), 4: (5, 21, 94)}[N]  # GeoW<N> in csrc/stp_wpe.cu
    a, b = build(N, *cur)
    print('current', cur, step_wavefronts(N, a, b))
