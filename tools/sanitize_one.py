"""One small u8 tensor-core build (racecheck triage)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

X = torch.from_numpy(datagen.make("sift", 2000, seed=3)).cuda()
K.knng_build(X, 16, 2, 8, 1)
torch.cuda.synchronize()
print("done")
