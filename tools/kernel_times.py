"""Per-kernel device time of one knng_build (CUDA events on the launch stream,
knng_set_timing) for several n / shapes -- where the step goes.
Usage: python tools/kernel_times.py [--shape sift] [--ns 1000000,2000000] [--iters 7]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

NAMES = ["k_init", "k_merge_sample", "k_scan_reduce", "k_scan_bsums", "k_scan_final", "k_rev_scatter",
         "k_rev_select", "k_join", "k_cand_scatter", "k_export", "k_check_u8", "k_to_u8", "k_normalize",
         "k_sqnorm_u8", "k_ggm_seed", "k_ggm_finalize", "k_order_colsum", "k_order_code", "k_order_scan",
         "k_order_scatter", "k_sqnorm_f32"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="sift")
    ap.add_argument("--ns", default="1000000,2000000,4000000")
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--metric", default="l2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for n in [int(x) for x in a.ns.split(",")]:
        X = torch.from_numpy(datagen.make(a.shape, n, seed=1, components=max(1000, n // 1000))).cuda()
        K.knng_build(X, a.k, a.iters, a.p, 42, a.metric)
        torch.cuda.synchronize()
        K.knng_set_timing(True)
        K.knng_reset_timing()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            ids, dists = K.knng_build(X, a.k, a.iters, a.p, 42, a.metric)
        e1.record()
        torch.cuda.synchronize()
        K.knng_set_timing(False)
        tot = e0.elapsed_time(e1) / a.reps
        per = {}
        for nm in NAMES:
            ms, cnt = K.knng_kernel_time(nm)
            if cnt:
                per[nm] = {"ms_per_build": round(ms / a.reps, 3), "launches": cnt // a.reps}
        st = K.knng_last_stats()
        print(json.dumps({"shape": a.shape, "n": n, "d": X.shape[1], "metric": a.metric,
                          "exact_u8": K.knng_get_option("last_exact_u8"), "ms_per_build": round(tot, 3),
                          "kernels": per, "dist_evals": sum(s["dist_evals"] for s in st),
                          "candidates": sum(s["candidates"] for s in st),
                          "recomputed": sum(s.get("recomputed", 0) for s in st)}), flush=True)
        del X, ids, dists
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
