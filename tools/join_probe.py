"""Float join role probe (profiling only, results are garbage under a probe):
time one k_join launch of the same mid-build state (iteration 2 of a
DEEP-shaped build) with parts of the warp-specialised pipeline disabled
(ws_probe bits: 1 consumers skip the math, 2 gathers skip the loads, 4 the
epilogue skips the filing).  Usage: python tools/join_probe.py [--n 1000000]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="deep")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--metric", default="l2")
ap.add_argument("--probes", default="0,1,2,4,6,7")
ap.add_argument("--opts", default="0,3")
ap.add_argument("--tword", type=int, default=2)
a = ap.parse_args()
X = datagen.make_device(a.shape, a.n, seed=1).cuda()
keys, flags = K.knng_debug_init(X, 32, 42, a.metric)
for t in range(a.tword):
    K.knng_debug_iterate(X, keys, flags, 16, t, 42, metric=a.metric)
k0, f0 = keys.clone(), flags.clone()
for o in a.opts.split(","):
    for pr in a.probes.split(","):
        K.knng_set_option("join_kernel", int(o))
        K.knng_set_option("ws_probe", int(pr))
        res = []
        for rep in range(3):
            keys.copy_(k0)
            flags.copy_(f0)
            K.knng_set_timing(True)
            K.knng_reset_timing()
            st = K.knng_debug_iterate(X, keys, flags, 16, a.tword, 42, metric=a.metric)
            K.knng_set_timing(False)
            ms, n = K.knng_kernel_time("k_join")
            res.append(ms / max(n, 1))
        print(f"{a.shape} n={a.n} {a.metric} join_kernel={o} probe={pr}: k_join {min(res):.3f} ms "
              f"(dist_evals {st['dist_evals']}, rows {st['rows']})", flush=True)
        if int(pr) & 32:
            # wait cycles per site, per warp of the role, as a fraction of the launch (3 reps summed)
            cyc = res[-1] * 1e-3 * 1.965e9 * 3
            names = {0: ("epi mfull", 4), 1: ("epi pfull", 4), 2: ("gather empty", 7), 4: ("gather mfull", 7),
                     5: ("lead mempty", 1), 7: ("cons mfull", 8), 8: ("cons pempty", 8), 20: ("cons full", 8),
                     10: ("lead publish", 1), 11: ("lead chunk", 1), 12: ("epi select", 4), 13: ("epi file", 4),
                     14: ("cons slab", 8), 15: ("cons minima", 8)}
            for i, (nm, w) in names.items():
                v = K.knng_get_option(f"ws_prof{i}")
                print(f"   {nm:14s} {v / (w * 148 * cyc):.3f}", flush=True)
K.knng_set_option("ws_probe", 0)
K.knng_set_option("join_kernel", 0)
