"""Diagnostic: k_join time per KNNG_JOIN_DBG mode (0 normal, 1 no tile math,
2 no gathers) on the C2 workload.  Results of modes 1/2 are garbage by design."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import datagen, paper_2103_15386_b200.knng as K
X = torch.from_numpy(datagen.make("sift", 1_000_000, seed=1)).cuda()
for _ in range(2):
    K.knng_build(X, 32, 8, 16, 42)
K.knng_set_timing(True); K.knng_reset_timing()
for _ in range(2):
    K.knng_build(X, 32, 8, 16, 42)
ms, n = K.knng_kernel_time("k_join")
print(os.environ.get("KNNG_JOIN_DBG", "0"), "k_join avg ms", ms / n)
'''
for mode in sys.argv[1:] or ["0", "1", "2"]:
    env = dict(os.environ, KNNG_JOIN_DBG=mode)
    subprocess.run([sys.executable, "-c", code], env=env, check=False)
