"""Text view of a per-launch step timeline (bench.py with GSB_TIMELINE=path; gsb_profile_timeline):
per stream, every launch with start / end (us from the first launch), and per-stream busy time
and gaps.  usage: python scripts/timeline.py path [max_us]"""
import sys
from collections import defaultdict

path = sys.argv[1]
lim = float(sys.argv[2]) if len(sys.argv) > 2 else 1e30
recs = []
for line in open(path):
    p = line.split()
    if len(p) != 4 or p[0] == "spin":
        continue
    recs.append((p[0], int(p[1]), float(p[2]), float(p[3])))
by = defaultdict(list)
for n, s, st, du in recs:
    if st <= lim:
        by[s].append((st, st + du, n))
for s in sorted(by):
    ev = sorted(by[s])
    busy = sum(e - b for b, e, _ in ev)
    span = ev[-1][1] - ev[0][0]
    print(f"== stream {s}: {len(ev)} launches, busy {busy:.1f} us of span {span:.1f} us "
          f"({ev[0][0]:.1f} .. {ev[-1][1]:.1f})")
    prev = None
    for b, e, n in ev:
        gap = "" if prev is None else f"  gap {b - prev:6.1f}"
        print(f"   {b:8.1f} {e:8.1f} {e - b:7.1f}  {n}{gap}")
        prev = e
