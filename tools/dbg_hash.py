import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, xxhash
import __graft_entry__; __graft_entry__.build()
import synth
from paper_1808_00117_b200 import crum
for P, nb in [(65536, 4 * 65536), (65536, 3 * 65536 + 1234), (2 << 20, 2 * (2 << 20)), (131072, 3 * 131072)]:
    g = crum.Context(0)
    t = torch.empty(nb, dtype=torch.uint8, device="cuda")
    crum.synth_fill(t, nb, synth.seed(1), 0)
    rid = g.register_region(t, nb, P, 1)
    g.sync_shadow()
    n = -(-nb // P)
    got = g.debug_export(rid, crum.EXPORT_HASHES, n)
    h = t.cpu().numpy()
    for i in range(n):
        seg = h[i * P:(i + 1) * P].tobytes(); seg += b"\0" * (P - len(seg))
        want = xxhash.xxh3_64_intdigest(seg)
        print(P, nb, i, hex(int(got[i])), hex(want), "OK" if int(got[i]) == want else "BAD")
