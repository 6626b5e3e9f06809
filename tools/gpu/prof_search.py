import cProfile, pstats, sys, os, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2509_24859_b200.planner import search
from paper_2509_24859_b200.profiling import boundary_costs, build_store
from paper_2509_24859_b200.workloads import instance
layers, cluster, model, rho, B, eps = instance('D1')
for i in range(3):
    st = build_store(layers, cluster, model, imbalance_ratio=rho); c = boundary_costs(layers, cluster)
    plan = search(st, c, B, epsilon=eps)
torch.cuda.synchronize()
pr = cProfile.Profile()
st = build_store(layers, cluster, model, imbalance_ratio=rho); c = boundary_costs(layers, cluster)
torch.cuda.synchronize()
pr.enable()
for i in range(5):
    plan = search(st, c, B, epsilon=eps)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(25)
