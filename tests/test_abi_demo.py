"""The C ABI from plain C (examples/abi_demo.c): compiles and links against
libhapt_b200.so with no Python/torch types involved (CPU), and on a GPU its
full-pool argmin plan equals the reference's search() plan (goldens)."""

import os
import shutil
import subprocess

import pytest

from helpers import expected, load_json, to_types

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
PKG = os.path.join(REPO, "paper_2509_24859_b200")
CUDA = "/usr/local/cuda"


def compile_demo(out_dir) -> str:
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no C compiler")
    exe = os.path.join(out_dir, "abi_demo")
    cmd = [gcc, "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror",
           f"-I{os.path.join(REPO, 'include')}", f"-I{CUDA}/include",
           os.path.join(REPO, "examples", "abi_demo.c"), "-o", exe,
           f"-L{PKG}", "-lhapt_b200", f"-L{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_demo_compiles_against_the_c_abi(tmp_path):
    if not os.path.exists(os.path.join(PKG, "libhapt_b200.so")):
        pytest.skip("library not built")
    compile_demo(str(tmp_path))


def write_instance(inst, path):
    from paper_2509_24859_b200.cluster import enumerate_submeshes

    layers, cluster, model, rho, B, eps = to_types(inst)
    lay = inst["layers"]
    meshes = list(cluster.meshes)
    opts = [(mi, sub.n, sub.m) for mi, mesh in enumerate(meshes)
            for sub in enumerate_submeshes(mesh)]
    cross = [cluster.cross_bandwidth(meshes[m].id, meshes[m + 1].id) if m + 1 < len(meshes)
             else 0.0 for m in range(len(meshes))]
    L = len(lay["flops"])
    vals = [L, len(meshes), len(opts), B]
    vals += lay["flops"] + lay["param_bytes"] + lay["boundary_bytes"] + lay["sig"]
    for m in meshes:
        vals += [m.hosts, m.devices_per_host, m.peak_flops, m.mem_device, m.intra_host_bw,
                 m.inter_host_bw]
    vals += cross
    vals += [o[1] for o in opts] + [o[2] for o in opts] + [o[0] for o in opts]
    vals += [cluster.cross_latency, model.beta, model.efficiency, model.alpha,
             model.replication, model.act_factor, rho,
             sum(float(x) for x in lay["flops"]),  # CPython sum, as the reference
             cluster.total_peak_flops, 1 if inst.get("dedup", True) else 0]
    with open(path, "w") as fh:
        fh.write(" ".join(repr(float(v)) if isinstance(v, float) else str(v) for v in vals))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["A", "C", "D1"])
def test_demo_plan_equals_reference(tmp_path, name):
    exe = compile_demo(str(tmp_path))
    inst = load_json(name)
    path = os.path.join(str(tmp_path), f"{name}.txt")
    write_instance(inst, path)
    r = subprocess.run([exe, path], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    tok = r.stdout.split()
    t_max, tstar, n = float(tok[0]), float(tok[1]), int(tok[3])
    plan = expected(name)["plan"]
    assert t_max == plan["t_max"] and tstar == plan["predicted_latency"]
    spans = [(int(tok[4 + 3 * i]), int(tok[5 + 3 * i])) for i in range(n)]
    assert spans == [tuple(s["layers"]) for s in plan["stages"]]
