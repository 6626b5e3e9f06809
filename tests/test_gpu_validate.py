"""GPU: the independent plan checker validate_plan (planner.py:615-670) on
plans that VIOLATE each constraint -- a stage gap, uncovered layers, mesh
order, devices left unused, a pruned span, a stage over t_max, memory over
budget, a comm-cost mismatch, comm over t_max -- returns exactly the
reference's violation messages (the unmodified reference, oracle/_ref,
checking the same plan dicts against its own store)."""

import copy

import pytest

from helpers import build, load_json, ref_types, reference_meshpipe

pytestmark = pytest.mark.gpu


def _mutations(d):
    """(name, mutated plan dict) pairs, each breaking one constraint."""
    S = len(d["stages"])
    out = []

    def mut(name, f):
        x = copy.deepcopy(d)
        f(x)
        out.append((name, x))

    mut("ok", lambda x: None)
    if S > 1:
        mut("gap", lambda x: x["stages"][1]["layers"].__setitem__(0, x["stages"][1]["layers"][0] + 1))
        mut("order", lambda x: (x["stages"][0].__setitem__("mesh", x["stages"][-1]["mesh"]),
                                x["stages"][-1].__setitem__("mesh", d["stages"][0]["mesh"])))
        mut("comm_mismatch", lambda x: x["boundaries"][0].__setitem__(
            "comm", x["boundaries"][0]["comm"] * 2 + 1e-3))
        mut("comm_over", lambda x: x["boundaries"][0].__setitem__("comm", x["t_max"] * 3))
    mut("uncovered", lambda x: x["stages"][-1]["layers"].__setitem__(
        1, x["stages"][-1]["layers"][1] - 1))
    mut("devices", lambda x: x["stages"][0].__setitem__("submesh", [1, 1]))
    mut("t_over", lambda x: x.__setitem__("t_max", x["t_max"] * 0.5))
    mut("memory", lambda x: x["stages"][0].__setitem__("dp_launch_bound", 10 ** 7))
    mut("pruned", lambda x: (x["stages"][0]["layers"].__setitem__(0, 1),
                             x["stages"][0]["layers"].__setitem__(1, x["stages"][-1]["layers"][1]),
                             x["stages"][0].__setitem__("submesh", [1, 1])))
    return out


@pytest.mark.parametrize("name", ["A", "B", "C"])
def test_validate_plan_violations_equal_reference(name):
    mp = reference_meshpipe()
    if mp is None:
        pytest.skip("oracle/_ref (the reference build) is not present")
    from paper_2509_24859_b200.planner import plan_from_dict, plan_to_dict, search, validate_plan

    inst = load_json(name)
    store, costs, cluster, B, eps = build(inst)
    plan = search(store, costs, B, epsilon=eps)
    rstore, rcosts, _, _ = ref_types(inst)
    seen = set()
    for what, d in _mutations(plan_to_dict(plan)):
        # errors (malformed plans, spans with no profile) must match too
        try:
            ours = validate_plan(plan_from_dict(d), store, costs, cluster)
        except Exception as exc:  # noqa: BLE001
            ours = (type(exc).__name__, str(exc))
        try:
            ref = mp.planner.validate_plan(mp.planner.plan_from_dict(d), rstore, rcosts,
                                           rstore.cluster)
        except Exception as exc:  # noqa: BLE001
            ref = (type(exc).__name__, str(exc))
        assert ours == ref, (name, what, ours, ref)
        if isinstance(ours, list):
            seen.update(m.split(":")[0].split(" ")[0] for m in ours)
        if what == "ok":
            assert ours == []
        elif isinstance(ours, list):
            assert ours, (name, what)  # every mutation is caught
    assert len(seen) >= 3
