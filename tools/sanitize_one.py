"""One small u8 tensor-core build and one restricted merge (racecheck
triage); prints a digest of the graphs so two builds can be compared."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

X = torch.from_numpy(datagen.make("sift", 2000, seed=3)).cuda()
ids, dists = K.knng_build(X, 16, 2, 8, 1)
ia, da = K.knng_build(X[:1000], 16, 2, 8, 2)
ib, db = K.knng_build(X[1000:], 16, 2, 8, 3)
mi, md = K.knng_merge(X[:1000], ia, da, X[1000:], ib, db, 16, 2, 8, seed=4)
torch.cuda.synchronize()
h = hashlib.sha256()
for t in (ids, dists, mi, md):
    h.update(t.cpu().numpy().tobytes())
print("graph digest", h.hexdigest())
