"""Per-task table of the row-stage trace of CTA 0 (output of trace_tc.py):
MMA1 issue, softmax start/end, MMA2 issue, epilogue start/end (set A, set B)."""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
ev = {}
for i, ln in enumerate(lines):
    m = re.match(r"cta 0 role (\d+):", ln)
    if m:
        role = int(m.group(1))
        ev[role] = [(int(t), float(x)) for t, x in re.findall(r"(\d+)@([\d.]+)", lines[i + 1])]
mma1 = [x for t, x in ev.get(1, []) if t == 11]
mma2 = [x for t, x in ev.get(1, []) if t == 12]
sm = {}
for role in (2,):   # softmax warp (quad 2)
    if role in ev:
        st = [x for t, x in ev[role] if t == 21]
        en = [x for t, x in ev[role] if t == 22]
        for k, (a, b) in enumerate(zip(st, en)):
            sm[k] = (a, b)
epA = {}
for role in (6,):
    if role in ev:
        st = [x for t, x in ev[role] if t == 31]
        en = [x for t, x in ev[role] if t == 32]
        for k, (a, b) in enumerate(zip(st, en)):
            epA[k] = (a, b)
epB = {}
for role in (10,):
    if role in ev:
        st = [x for t, x in ev[role] if t == 31]
        en = [x for t, x in ev[role] if t == 32]
        for k, (a, b) in enumerate(zip(st, en)):
            epB[k] = (a, b)
print(" t   mma1   sm_st  sm_en   mma2   epA_st epA_en  epB_st epB_en")
for t in range(len(mma1)):
    f = lambda d: ("%6.2f %6.2f" % d[t]) if t in d else "   -      -  "
    print(f"{t:2d} {mma1[t]:6.2f}  {f(sm)}  {mma2[t] if t < len(mma2) else 0:6.2f}  {f(epA)}  {f(epB)}")
