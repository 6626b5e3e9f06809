"""B200-native HAPT planner hot path (arXiv 2509.24859).

Drop-in for the planner/scheduler entry points of the reference package
`meshpipe` (SPEC.md module interfaces): cost tables (K1), the batched
stage-partition DP over every t_max candidate (K2) and the 1F1B schedule
evaluation (K3) run as sm_100a kernels in libhapt_b200.so (C ABI,
include/hapt_b200.h).  PyTorch only provides device memory, streams and
torch.distributed (NCCL) for sharding candidates across GPUs.

Modules mirror the reference layout: cluster, model_graph (input types),
profiling, planner, scheduling, simulation, _core (dp_sweep operator);
distributed adds the multi-GPU candidate sharding.
"""

BACKEND = "cuda"
__version__ = "0.1.0"
__all__ = ["BACKEND", "__version__"]
