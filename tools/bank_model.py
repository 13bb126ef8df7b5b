"""Shared-memory bank model of the bipartite line-pass kernel (stp_pass.cu, GeoB): counts the
wavefronts of every pass's source-line loads and target accesses for a given row / plane / field
padding and searches the padding.  64-bit accesses: per half-warp, max multiplicity of the bank
pair (address mod 16 doubles) over distinct addresses; 128-bit: per quarter-warp (address/2 mod 8).
Usage: python tools/bank_model.py N"""
import itertools, sys
def wf64(addrs):
    tot = 0
    for h in (addrs[:16], addrs[16:]):
        h = [a for a in h if a is not None]
        if not h: continue
        cnt = {}
        for a in set(h): cnt[a % 16] = cnt.get(a % 16, 0) + 1
        tot += max(cnt.values())
    return tot
def wf128(addrs):
    tot = 0
    for qq in range(4):
        h = [a for a in addrs[qq*8:qq*8+8] if a is not None]
        if not h: continue
        cnt = {}
        for a in set(h): cnt[(a // 2) % 8] = cnt.get((a // 2) % 8, 0) + 1
        tot += max(cnt.values())
    return tot
PASSES = {
  'Vx': ([0,3,4], [[9],[10],[11]], 0), 'Vy': ([3,1,5], [[9],[10],[11]], 1), 'Vz': ([4,5,2], [[9],[10],[11]], 2),
  'Sx': ([6,7,8], [[0,1,2],[3],[4]], 0), 'Sy': ([7,6,8], [[0,1,2],[3],[5]], 1), 'Sz': ([8,6,7], [[0,1,2],[4,3],[5]], 2)}
def cost(N, RS, PL, VS, lanemap, x128, ideal=False):
    # lanemap: list over threads of (slot, line) or None
    total = 0
    nw = (len(lanemap) + 31) // 32
    for name, (src, tgt, d) in PASSES.items():
        for w in range(nw):
            lanes = []
            for lane in range(32):
                t = w * 32 + lane
                x = lanemap[t] if t < len(lanemap) else None
                if x is None: lanes.append(None); continue
                slot, line = x
                la, lb = divmod(line, N)
                start = la*PL + lb*RS if d == 0 else la*PL + lb if d == 1 else la*RS + lb
                lanes.append((slot, start))
            use128 = x128 and d == 0
            def W(ad):
                if ideal:
                    if use128: return sum(1 for q in range(4) if any(a is not None for a in ad[q*8:q*8+8]))
                    return sum(1 for h in (ad[:16], ad[16:]) if any(a is not None for a in h))
                return wf128(ad) if use128 else wf64(ad)
            reps = (N + 1) // 2 if use128 else N
            total += reps * W([None if x is None else src[x[0]]*VS + x[1] for x in lanes])
            for k in range(3):
                ad = [None if x is None or k >= len(tgt[x[0]]) else tgt[x[0]][k]*VS + x[1] for x in lanes]
                if all(a is None for a in ad): continue
                total += reps * W(ad) * (1 if d == 0 else 2)
    return total
import sys
N = int(sys.argv[1]); L = N*N
def cost_s(N, RS, PL, VS, lanemap, x128, swap):
    total = 0
    nw = (len(lanemap) + 31) // 32
    for name, (src, tgt, d) in PASSES.items():
        for w in range(nw):
            lanes = []
            for lane in range(32):
                t = w * 32 + lane
                x = lanemap[t] if t < len(lanemap) else None
                if x is None: lanes.append(None); continue
                slot, line = x
                la, lb = divmod(line, N)
                if swap[d]: la, lb = lb, la
                start = la*PL + lb*RS if d == 0 else la*PL + lb if d == 1 else la*RS + lb
                lanes.append((slot, start))
            use128 = x128 and d == 0
            W = wf128 if use128 else wf64
            reps = (N + 1) // 2 if use128 else N
            total += reps * W([None if x is None else src[x[0]]*VS + x[1] for x in lanes])
            for k in range(3):
                ad = [None if x is None or k >= len(tgt[x[0]]) else tgt[x[0]][k]*VS + x[1] for x in lanes]
                if all(a is None for a in ad): continue
                total += reps * W(ad) * (1 if d == 0 else 2)
    return total
m_cur = [(t // L, t % L) if t < 3 * L else None for t in range(((3*L+31)//32)*32)]
res = []
RSs = (N, N+1) if N % 2 == 0 else (N, N+1, N+2)
for RS in RSs:
  for PL in range(N*RS, N*RS+16):
    for VS in range(N*PL, N*PL+16, 1):
      if 12*VS*8 > 113*1024 and N == 10: continue
      for swap in itertools.product((0,1), repeat=3):
        for x128 in (False, True):
          if x128 and (RS % 2 or PL % 2 or N % 2): continue
          res.append((cost_s(N, RS, PL, VS, m_cur, x128, swap), RS, PL, VS, x128, swap))
res.sort(); print(res[:8])
