#!/usr/bin/env python3
"""Bank model of the warp-per-element kernel (stp_wpe): shared-memory wavefronts of the CK-step
loads/stores for a layout [k3][k2][s][k1] with strides (1, 6, S2, S3) and a lane -> task map.
64-bit accesses: a warp instruction is served per half-warp; wavefronts = max distinct addresses
per 8-byte bank (16 banks)."""
import itertools, sys
N = 6
def wf(addrs):  # addrs: list of (lane, addr) active
    tot = 0
    for h in (0, 1):
        banks = {}
        for lane, a in addrs:
            if lane // 16 == h:
                banks.setdefault(a % 16, set()).add(a)
        if banks:
            tot += max(len(v) for v in banks.values())
    return tot

def strides(S2, S3):
    return {'x': 1, 'y': S2, 'z': S3}

def model(S2, S3, tasksA, tasksB, verbose=False):
    st = strides(S2, S3)
    total = 0
    ideal = 0
    for tasks in (tasksA, tasksB):
        # each task: list of terms (field, d, o, fixed_dir, fixed_idx); loads per (j, l)
        for term in (0, 1):
            for j in range(N):
                for l in range(N):
                    addrs = []
                    for lane, t in enumerate(tasks):
                        if t is None or t[term] is None: continue
                        f, d, o, fd, fi = t[term]
                        addrs.append((lane, 6 * f + l * st[d] + j * st[o] + fi * st[fd]))
                    if addrs:
                        total += wf(addrs); ideal += (len(addrs) + 15) // 16
        # stores of the result (dst field, tile dirs) : index (i, j) over the tile of term 0 dst
        for i in range(N):
            for j in range(N):
                for which in (2, 3):
                    addrs = []
                    for lane, t in enumerate(tasks):
                        if t is None or len(t) <= which or t[which] is None: continue
                        f, d, o, fd, fi = t[which]
                        addrs.append((lane, 6 * f + i * st[d] + j * st[o] + fi * st[fd]))
                    if addrs:
                        total += wf(addrs); ideal += (len(addrs) + 15) // 16
    return total, ideal

SXX, SYY, SZZ, SXY, SXZ, SYZ, U, V, W = range(9)
def build(part_orient='x', orderA=None):
    # phase A: shear tasks and partial pairs.  task = (termA, termB, dst1, dst2)
    A = []
    for k in range(N): A.append(((V, 'x', 'y', 'z', k), (U, 'y', 'x', 'z', k), (SXY, 'x', 'y', 'z', k), None))
    for k in range(N): A.append(((W, 'x', 'z', 'y', k), (U, 'z', 'x', 'y', k), (SXZ, 'x', 'z', 'y', k), None))
    for k in range(N): A.append(((W, 'y', 'z', 'x', k), (V, 'z', 'y', 'x', k), (SYZ, 'y', 'z', 'x', k), None))
    # partial units: z-derivative of src -> dst slot, tile (z, o) at fixed third dir
    units = []
    for src, dst in ((SXZ, U), (SYZ, V), (SZZ, W), (W, SZZ)):
        for k in range(N):
            o, fd = ('x', 'y') if part_orient == 'x' else ('y', 'x')
            units.append(((src, 'z', o, fd, k), (dst, 'z', o, fd, k)))
    return A, units

def phaseB():
    B = []
    for k in range(N): B.append(((SXX, 'x', 'y', 'z', k), (SXY, 'y', 'x', 'z', k), (U, 'x', 'y', 'z', k), None))
    for k in range(N): B.append(((SXY, 'x', 'y', 'z', k), (SYY, 'y', 'x', 'z', k), (V, 'x', 'y', 'z', k), None))
    for k in range(N): B.append(((SXZ, 'x', 'y', 'z', k), (SYZ, 'y', 'x', 'z', k), (W, 'x', 'y', 'z', k), None))
    for k in range(N): B.append(((U, 'x', 'y', 'z', k), (V, 'y', 'x', 'z', k), (SXX, 'x', 'y', 'z', k), (SYY, 'x', 'y', 'z', k)))
    return B

if __name__ == '__main__':
    best = []
    for po in ('x', 'y'):
        A, units = build(po)
        # pairings of the 24 partial units onto 12 lanes: (unit i, unit i+12) or (2i, 2i+1)
        for pairing in ('half', 'adjacent', 'stride6'):
            if pairing == 'half': pairs = [(units[i], units[i + 12]) for i in range(12)]
            elif pairing == 'adjacent': pairs = [(units[2 * i], units[2 * i + 1]) for i in range(12)]
            else: pairs = [(units[(i % 6) + 12 * (i // 6)], units[(i % 6) + 12 * (i // 6) + 6]) for i in range(12)]
            tA = list(A) + [(p[0][0], p[1][0], p[0][1], p[1][1]) for p in pairs]
            tB = phaseB()
            for S2 in range(54, 72, 2):
                for p3 in range(0, 34, 2):
                    S3 = 6 * S2 + p3
                    t, i = model(S2, S3, tA, tB)
                    best.append((t, i, po, pairing, S2, S3))
    best.sort()
    for b in best[:15]: print(b)
    print('compact', [b for b in best if b[4] == 54 and b[5] == 324])
