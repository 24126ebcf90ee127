import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import synth
from tests.gpu_pair import Pair
from tests.test_gpu_parity import MIXED
from paper_1808_00117_b200 import crum
p = Pair(MIXED, synth.seed(10))
print("detect0", np.array_equal(p.g.debug_detect(p.N), p.oracle_flags()))
print("sync", p.g.sync_shadow(), p.o.sync_shadow(), p.N)
for (nb, P, mode), ro, rg in zip(p.specs, p.rid_o, p.rid_g):
    n = synth.n_pages(nb, P)
    fo, fg = p.o.force_bits(ro), p.g.debug_export(rg, crum.EXPORT_FORCE, n)
    print(nb, P, mode, "force", np.array_equal(fo, fg), fo.sum(), fg.sum())
    if mode == 1:
        ho, hg = p.o.hashes(ro), p.g.debug_export(rg, crum.EXPORT_HASHES, n)
        print("   hashes", np.array_equal(ho, hg), [i for i in range(n) if ho[i] != hg[i]][:10])
    else:
        mo, mg = p.o.mirror(ro), p.g.debug_export(rg, crum.EXPORT_MIRROR, nb)
        bad = np.flatnonzero(mo != mg)
        print("   mirror", np.array_equal(mo, mg), bad[:5], len(bad))
