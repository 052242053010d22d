"""Critical-path view of one c3 factorization from the library's per-launch
event timeline (randutv_profile_timeline): per stream, busy time by class and
the idle gaps of the main stream (host synchronisation bubbles, launch gaps).
usage: python tools/timeline.py [config] [scale]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
At, c = testmat.device_config(name, scale=scale)
A = At.t()
m, n = A.shape
T = P.empty_cm(m, n)
for _ in range(2):
    P.randutv(A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False, out=(None, T, None))
torch.cuda.synchronize()
P.profile_begin()
_, _, _, info = P.randutv(A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False, out=(None, T, None))
P.profile_end()
tl = P.profile_timeline()
end = max(e for _, _, _, e in tl)
print(f"{name} {m}x{n}: profiled factorization spans {end:.2f} ms, {len(tl)} launches, max_sweeps={info.max_sweeps}")
by_stream = collections.defaultdict(list)
for cls, s, a, e in tl:
    by_stream[s].append((a, e, cls))
for s, ev in sorted(by_stream.items()):
    ev.sort()
    busy = collections.Counter()
    for a, e, cls in ev:
        busy[cls] += e - a
    # union of intervals
    tot, cur_a, cur_e = 0.0, None, None
    gaps = []
    for a, e, _ in ev:
        if cur_e is None or a > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_a
                gaps.append(a - cur_e)
            cur_a, cur_e = a, e
        else:
            cur_e = max(cur_e, e)
    tot += cur_e - cur_a
    print(f"stream {s}: first {ev[0][0]:.2f} ms last {cur_e:.2f} ms busy {tot:.2f} ms; "
          f"idle gaps {sum(gaps):.2f} ms in {len(gaps)} gaps (>20us: {sum(g for g in gaps if g > 0.02):.2f} ms)")
    for cls, v in busy.most_common():
        print(f"    {cls:18s} {v:8.2f} ms")
out = os.environ.get("TIMELINE_OUT")
if out:  # raw per-launch records for offline analysis
    import json
    with open(out, "w") as f:
        json.dump(tl, f)
