"""knng_merge wall time vs its kernels: with / without a caller workspace and
per-kernel timing (where do the gaps between kernels come from)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

X = torch.from_numpy(datagen.make("sift", 1_000_000, seed=1)).cuda()
h = 500_000
ia, da = K.knng_build(X[:h], 32, 7, 16, 42)
ib, db = K.knng_build(X[h:], 32, 7, 16, 43)
ws = torch.empty(K.lib().knng_merge_workspace_bytes(K.KNNG_F32, h, h, 128, 32, 16, 0), dtype=torch.uint8,
                 device="cuda")
for use_ws in (False, True):
    for timing in (False, True):
        K.knng_set_timing(timing)
        f = lambda: K.knng_merge(X[:h], ia, da, X[h:], ib, db, 32, 6, 16, seed=42,  # noqa: E731
                                 workspace=ws if use_ws else None)
        f()
        torch.cuda.synchronize()
        K.knng_reset_timing()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 3 * 1e3
        print(f"workspace={use_ws} timing={timing}: events {e0.elapsed_time(e1) / 3:.2f} ms, wall {wall:.2f} ms",
              flush=True)
K.knng_set_timing(False)
