python tools/build_ab.py 2 1.0 "MRPT_PROJ_D64=1" "MRPT_PROJ_D64=1"
python - <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import paper_1509_06957_b200 as mrpt
from paper_1509_06957_b200 import workloads
X, Q, p = workloads.generate(2)
warm = torch.randn(512, X.shape[1], device="cuda")
mrpt.grow_trees(warm, 2, 3, seed=1)
Xd = torch.from_numpy(X).cuda(); torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter(); idx = mrpt.grow_trees(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=0); torch.cuda.synchronize(); print("build", time.perf_counter() - t0)
PY
