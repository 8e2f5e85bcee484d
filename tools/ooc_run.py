"""Out-of-memory all-pairs construction (knng_build_ooc) on a
synthetic set held in host memory: wall time of the call (host buffers in and
out, copies overlapped with the merges), recall@10 on 10k sampled nodes.

  python tools/ooc_run.py --shape sift --n 8000000 --shards 8 --k 32 --p 16"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="sift")
    ap.add_argument("--n", type=int, default=8_000_000)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--merge-iters", type=int, default=6)
    ap.add_argument("--components", type=int, default=None)
    ap.add_argument("--u8", action="store_true", help="store SIFT-shaped rows as uint8 (C5 style)")
    a = ap.parse_args()
    Xd = datagen.make_device(a.shape, a.n, seed=3, components=a.components)
    if a.u8:
        Xd = Xd.to(torch.uint8)
    Xh = Xd.cpu().numpy()
    Xh = np.ascontiguousarray(Xh)
    ids = np.empty((a.n, a.k), np.uint32)
    dists = np.empty((a.n, a.k), np.float32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K.knng_build_ooc(Xh, a.k, a.iters, a.merge_iters, a.p, a.shards, seed=42, out_ids=ids, out_dists=dists)
    wall = time.perf_counter() - t0
    nodes = datagen.sample_nodes(a.n, 10000)
    q = torch.from_numpy(nodes).cuda()
    _, td = K.knng_bruteforce(Xd, q, 10)
    t10 = td.cpu().numpy()[:, 9]
    rec = float((dists[nodes, :10] <= t10[:, None]).sum()) / (10 * len(nodes))
    out = {"workload": f"{a.shape}-shaped {a.n} x {Xh.shape[1]} {'u8' if a.u8 else 'f32'} in host memory, "
                       f"{a.shards} shards, all {a.shards * (a.shards - 1) // 2} pairs merged",
           "n": a.n, "shards": a.shards, "k": a.k, "p": a.p, "iters": a.iters, "merge_iters": a.merge_iters,
           "seconds": wall, "recall_at_10": rec, "recall_nodes": len(nodes),
           "host_bytes_in": int(Xh.nbytes), "host_bytes_out": int(ids.nbytes + dists.nbytes)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
