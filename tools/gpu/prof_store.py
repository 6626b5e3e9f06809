"""Host profile of build_store + boundary_costs + sweep_pool (the bench's e2e path), D1."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2509_24859_b200.planner import sweep_pool  # noqa: E402
from paper_2509_24859_b200.profiling import boundary_costs, build_store  # noqa: E402
from paper_2509_24859_b200.workloads import instance  # noqa: E402

layers, cluster, model, rho, B, eps = instance(sys.argv[1] if len(sys.argv) > 1 else "D1")
for _ in range(5):
    st = build_store(layers, cluster, model, imbalance_ratio=rho)
    sweep_pool(st, boundary_costs(layers, cluster), B)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    st = build_store(layers, cluster, model, imbalance_ratio=rho)
    c = boundary_costs(layers, cluster)
    sweep_pool(st, c, B)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
