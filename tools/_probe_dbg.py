import os, sys, subprocess, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2509_24859_b200.planner import DpTables
from paper_2509_24859_b200.profiling import boundary_costs, build_store
from paper_2509_24859_b200.workloads import instance
name = sys.argv[1]
layers, cluster, model, rho, B, eps = instance(name)
store = build_store(layers, cluster, model, imbalance_ratio=rho)
tables = DpTables(store, boundary_costs(layers, cluster))
pool = np.asarray(store.feasible_t_values())
sw = tables.sweeper
ftop, states = sw.sweep_device(torch.from_numpy(pool).cuda())
np.save(f"/tmp/ftop_{os.environ.get('HAPT_PROBE','1')}.npy", ftop.cpu().numpy())
np.save(f"/tmp/st_{os.environ.get('HAPT_PROBE','1')}.npy", states.cpu().numpy())
# single candidate full tables for the first few candidates
