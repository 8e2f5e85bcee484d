"""Small builds/merges on every join path, for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

Xs = torch.from_numpy(datagen.make("sift", 3000, seed=3)).cuda()      # exact-u8 tensor-core join (TMA)
Xd = torch.from_numpy(datagen.make("deep", 3000, seed=3)).cuda()      # float join
for jk in [0, 2, 3]:
    K.knng_set_option("join_kernel", jk)
    K.knng_build(Xs, 16, 3, 8, 1)
    K.knng_build(Xd, 16, 3, 8, 1)
    K.knng_build(Xd, 16, 3, 8, 1, "cosine")
    ia, da = K.knng_build(Xs[:1500], 16, 3, 8, 2)
    ib, db = K.knng_build(Xs[1500:], 16, 3, 8, 3)
    K.knng_merge(Xs[:1500], ia, da, Xs[1500:], ib, db, 16, 2, 8, seed=4)
K.knng_set_option("join_kernel", 0)
torch.cuda.synchronize()
print("sanitize workload done")
