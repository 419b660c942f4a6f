"""File-format interop: allocation.json, assignment.json and
profiles.json written by the reference library load unchanged here, files
written here load in the reference and are byte-identical to the reference's
own output, and malformed files fail with the reference's messages
(allocator.cpp:223-275, partitioner.cpp:268-336, profiler.cpp:300-383)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2603_10353_b200 as P
from oracle import oracle as O
from paper_2603_10353_b200 import formats as F

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")


def _curves(seed=3, hq=6, n_k=512, stride=64):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((hq, 4, 128)).astype(np.float32) * rng.uniform(0.05, 0.5, (hq, 1, 1)).astype(np.float32)
    k = rng.standard_normal((2, n_k, 128)).astype(np.float32)
    return P.profile_curves(O.f32_to_bf16_bits(q), O.f32_to_bf16_bits(k), P.default_budget_grid(n_k, stride))


def _read(p):
    with open(p) as f:
        return f.read()


# ------------------------------------------------------------ round trips --

def test_allocation_round_trip(tmp_path):
    curves = _curves()
    alloc = P.maxmin_allocate(curves, 6 * 200, quantum=64, floor=64)
    p = str(tmp_path / "allocation.json")
    F.save_allocation(p, alloc.budgets, alloc.total, alloc.floor, heads=[(3, h) for h in range(6)])
    a = F.load_allocation(p)
    assert np.array_equal(a.budgets, alloc.budgets) and a.total == alloc.total and a.floor == alloc.floor
    assert a.heads == [(3, h) for h in range(6)]


def test_assignment_and_profiles_round_trip(tmp_path):
    budgets = np.array([900, 128, 640, 300, 128, 1000], np.int64)
    dev = P.greedy_assign(budgets, 3)
    rep = P.imbalance(budgets, dev, 3)
    p = str(tmp_path / "assignment.json")
    F.save_assignment(p, dev, 3, rep.loads, rep.imbalance)
    a = F.load_assignment(p)
    assert np.array_equal(a.device_of_head, dev) and a.devices == 3
    assert np.array_equal(a.loads, rep.loads) and a.imbalance == rep.imbalance
    curves = _curves()
    p = str(tmp_path / "profiles.json")
    F.save_profiles(p, curves)
    lp = F.load_profiles(p)
    assert lp.policy == "per_query_topk" and lp.context_length == 512
    for c, d in zip(curves, lp.curves):
        assert np.array_equal(c.budgets, d.budgets) and np.array_equal(c.recovery, d.recovery)


# ------------------------------------------------- against the reference --

@needs_ref
def test_reference_written_files_load_here(tmp_path):
    curves = _curves(7)
    alloc = P.maxmin_allocate(curves, 6 * 256, quantum=64, floor=128)
    pa = str(tmp_path / "a.json")
    O.ref.save_allocation(pa, alloc.budgets, alloc.total, alloc.floor, heads=[(1, h) for h in range(6)])
    la = F.load_allocation(pa)
    assert np.array_equal(la.budgets, alloc.budgets) and la.heads == [(1, h) for h in range(6)]

    dev = P.greedy_assign(alloc.budgets, 4)
    rep = P.imbalance(alloc.budgets, dev, 4)
    ps = str(tmp_path / "s.json")
    O.ref.save_assignment(ps, dev, 4, rep.loads, rep.imbalance)
    ls = F.load_assignment(ps)
    assert np.array_equal(ls.device_of_head, dev) and np.array_equal(ls.loads, rep.loads)
    assert ls.imbalance == rep.imbalance and ls.total == int(rep.loads.sum())

    pp = str(tmp_path / "p.json")
    O.ref.save_profiles(pp, [c.budgets for c in curves], [c.recovery for c in curves], 512,
                        request="req-1", task="needle")
    lp = F.load_profiles(pp)
    assert lp.provenance[0] == ("req-1", "needle")
    for c, d in zip(curves, lp.curves):  # fp64 survives the text round trip exactly
        assert np.array_equal(c.budgets, d.budgets) and np.array_equal(c.recovery, d.recovery)


@needs_ref
def test_files_written_here_are_byte_identical_and_load_in_reference(tmp_path):
    curves = _curves(9)
    alloc = P.maxmin_allocate(curves, 6 * 256, quantum=64, floor=128)
    ours, theirs = str(tmp_path / "ours.json"), str(tmp_path / "theirs.json")
    F.save_allocation(ours, alloc.budgets, alloc.total, alloc.floor)
    O.ref.save_allocation(theirs, alloc.budgets, alloc.total, alloc.floor)
    assert _read(ours) == _read(theirs)
    b, heads, tot, fl = O.ref.load_allocation(ours)
    assert np.array_equal(b, alloc.budgets) and tot == alloc.total

    dev = P.greedy_assign(alloc.budgets, 4)
    rep = P.imbalance(alloc.budgets, dev, 4)
    F.save_assignment(ours, dev, 4, rep.loads, rep.imbalance)
    O.ref.save_assignment(theirs, dev, 4, rep.loads, rep.imbalance)
    assert _read(ours) == _read(theirs)
    d2, _, nd, loads, _, imb = O.ref.load_assignment(ours)
    assert np.array_equal(d2, dev) and nd == 4 and imb == rep.imbalance

    F.save_profiles(ours, curves, request="r", task="t")
    O.ref.save_profiles(theirs, [c.budgets for c in curves], [c.recovery for c in curves], 512,
                        request="r", task="t")
    assert _read(ours) == _read(theirs)
    got, _, n_k, kind, req, task = O.ref.load_profiles(ours)
    assert n_k == 512 and kind == 0 and (req, task) == ("r", "t")
    for c, (b, r) in zip(curves, got):
        assert np.array_equal(c.budgets, b) and np.array_equal(c.recovery, r)


def _mutations():
    good_a = {"version": 1, "total": 384, "floor": 128,
              "budgets": [{"layer": 0, "head": 0, "budget": 128}, {"layer": 0, "head": 1, "budget": 256}]}
    good_s = {"version": 1, "devices": 2, "imbalance": 1.3333333333333333, "loads": [256, 128],
              "assignment": [{"layer": 0, "head": 0, "device": 1}, {"layer": 0, "head": 1, "device": 0}]}
    good_p = {"version": 1, "policy": "per_query_topk", "context_length": 100,
              "profiles": [{"layer": 0, "head": 0, "points": [[0, 0.0], [50, 0.7], [100, 1.0]],
                            "provenance": {"request": "r", "task": "t"}}]}

    def m(base, f):
        d = json.loads(json.dumps(base))
        f(d)
        return d

    A, S, Pf = "allocation", "assignment", "profiles"
    return [
        (A, m(good_a, lambda d: d.update(extra=1))),
        (A, m(good_a, lambda d: d.pop("floor"))),
        (A, m(good_a, lambda d: d.update(version=2))),
        (A, m(good_a, lambda d: d.update(total="384"))),
        (A, m(good_a, lambda d: d.update(budgets=[]))),
        (A, m(good_a, lambda d: d["budgets"][1].update(budget=64))),
        (A, m(good_a, lambda d: d.update(total=999))),
        (A, m(good_a, lambda d: d["budgets"][0].update(budget=128.0))),
        (A, m(good_a, lambda d: d["budgets"][0].update(weight=1))),
        (S, m(good_s, lambda d: d["assignment"][1].update(head=0))),
        (S, m(good_s, lambda d: d["assignment"][1].update(device=2))),
        (S, m(good_s, lambda d: d.update(loads=[1]))),
        (S, m(good_s, lambda d: d.update(loads=[1, 2.5]))),
        (S, m(good_s, lambda d: d.update(imbalance=0.5))),
        (S, m(good_s, lambda d: d.update(imbalance="x"))),
        (S, m(good_s, lambda d: d.update(devices=0))),
        (Pf, m(good_p, lambda d: d["profiles"][0].update(points=[[0, 0.0], [60, 0.5]]))),
        (Pf, m(good_p, lambda d: d["profiles"][0].update(points=[[0, 0.0], [50, 0.9], [40, 0.95], [100, 1.0]]))),
        (Pf, m(good_p, lambda d: d["profiles"][0].update(points=[[0, 0.0], [50, 0.9], [60, 0.5], [100, 1.0]]))),
        (Pf, m(good_p, lambda d: d["profiles"][0].update(points=[[0, 0.0], [100, 0.9]]))),
        (Pf, m(good_p, lambda d: d["profiles"][0].update(points=[[0, 0.0], [100, "1"]]))),
        (Pf, m(good_p, lambda d: d["profiles"][0].update(points=[[0.5, 0.0], [100, 1.0]]))),
        (Pf, m(good_p, lambda d: d["profiles"][0]["provenance"].update(task=""))),
        (Pf, m(good_p, lambda d: d["profiles"][0]["provenance"].update(user="x"))),
        (Pf, m(good_p, lambda d: d.update(profiles=[]))),
        (Pf, m(good_p, lambda d: d.update(context_length=1.5))),
    ]


@needs_ref
@pytest.mark.parametrize("case", range(len(_mutations())))
def test_malformed_files_fail_with_reference_messages(tmp_path, case):
    kind, doc = _mutations()[case]
    p = str(tmp_path / f"{kind}.json")
    with open(p, "w") as f:
        json.dump(doc, f)
    loaders = {"allocation": (F.load_allocation, O.ref.load_allocation),
               "assignment": (F.load_assignment, O.ref.load_assignment),
               "profiles": (F.load_profiles, O.ref.load_profiles)}
    ours, theirs = loaders[kind]
    with pytest.raises(O.ReferenceError) as ref_err:
        theirs(p)
    with pytest.raises(P.ShplbError) as our_err:
        ours(p)
    assert str(our_err.value) == str(ref_err.value)


def test_missing_file_and_bad_policy(tmp_path):
    with pytest.raises(P.ShplbRuntimeError, match="cannot open"):
        F.load_allocation(str(tmp_path / "nope.json"))
    p = str(tmp_path / "p.json")
    with open(p, "w") as f:
        json.dump({"version": 1, "policy": "top_p", "context_length": 4,
                   "profiles": [{"layer": 0, "head": 0, "points": [[4, 1.0]],
                                 "provenance": {"request": "r", "task": "t"}}]}, f)
    with pytest.raises(P.InvalidArgument, match='unknown selection policy "top_p"'):
        F.load_profiles(p)
    assert os.path.exists(p)


# ---------------------------------------------------------------------------
# stability_score (profiler.cpp:233-292): the paper's cross-request stability
# ---------------------------------------------------------------------------

def _step_curve(n_k, knee):
    """Recovery 0 below `knee` tokens, 1 from it on (test_profiler.cpp step_curve)."""
    b = sorted({0, knee, n_k})
    return P.RecoveryCurve(np.array(b, np.int64), np.array([0.0 if x < knee else 1.0 for x in b]), n_k)


def _group(curves, request, heads=None):
    from paper_2603_10353_b200.formats import LoadedProfiles
    heads = heads or [(0, h) for h in range(len(curves))]
    return LoadedProfiles(curves, heads, "per_query_topk", curves[0].context_length,
                          [(request, "parity")] * len(curves))


def test_stability_identical_and_rescaled_requests():
    """'stability is 1 for identical and for rescaled requests' (test_profiler.cpp:167-178)."""
    from paper_2603_10353_b200.formats import stability_score
    base = _group([_step_curve(1024, 64), _step_curve(1024, 256), _step_curve(1024, 512)], "req-a")
    assert stability_score([base, base, base], 0.9) == pytest.approx(1.0, abs=1e-12)
    doubled = _group([_step_curve(2048, 128), _step_curve(2048, 512), _step_curve(2048, 1024)], "req-b")
    assert stability_score([base, doubled], 0.9) == pytest.approx(1.0, abs=1e-12)
    assert stability_score([base, doubled], 0.9, "sum") == pytest.approx(1.0, abs=1e-12)


def test_stability_rejects_degenerate_and_mismatched_groups():
    """test_profiler.cpp:208-221, with the reference's messages."""
    from paper_2603_10353_b200.formats import stability_score
    degenerate = _group([_step_curve(64, 16), _step_curve(64, 16)], "flat-request")
    good = _group([_step_curve(64, 8), _step_curve(64, 32)], "ok-request")
    with pytest.raises(P.InvalidArgument, match="flat-request: budget vector has zero variance"):
        stability_score([good, degenerate], 0.9)
    with pytest.raises(P.InvalidArgument, match="needs at least 2 calibration requests"):
        stability_score([good], 0.9)
    other = _group([_step_curve(64, 8), _step_curve(64, 32)], "req-x", heads=[(0, 0), (0, 5)])
    with pytest.raises(P.InvalidArgument, match="req-x: head set differs from the first request"):
        stability_score([good, other], 0.9)


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built")
def test_stability_matches_reference_on_profiled_requests():
    """Three calibration 'requests' (different query rows of one synthetic head
    set), profiled here: the score equals the reference's stability_score."""
    from paper_2603_10353_b200.formats import stability_score
    rng = np.random.default_rng(17)
    k = O.f32_to_bf16_bits(rng.standard_normal((2, 512, 128)).astype(np.float32))
    temps = rng.uniform(0.05, 0.6, (8, 1, 1)).astype(np.float32)
    groups, ref_groups = [], []
    for req in range(3):
        q = O.f32_to_bf16_bits(rng.standard_normal((8, 6, 128)).astype(np.float32) * temps)
        curves = P.profile_curves(q, k, P.default_budget_grid(512, 8))
        heads = [(1, h) for h in range(8)][::-1]  # out of order on purpose: sorted by id inside
        curves = curves[::-1]
        groups.append(_group(curves, f"request-{req}", heads))
        ref_groups.append((f"request-{req}", heads, curves))
    for p in (0.5, 0.9):
        for norm in ("max", "sum"):
            ours = stability_score(groups, p, norm)
            ref = O.ref.stability_score(ref_groups, p, norm)
            assert ours == pytest.approx(ref, abs=1e-12), (p, norm, ours, ref)


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built")
def test_budget_for_recovery_matches_reference_on_random_curves():
    rng = np.random.default_rng(4)
    for _ in range(50):
        n_k = int(rng.integers(2, 400))
        pts = np.unique(np.concatenate([[n_k], rng.integers(0, n_k, rng.integers(1, 20))]))
        rec = np.sort(rng.uniform(0, 1, pts.size))
        rec[-1] = 1.0
        c = P.RecoveryCurve(pts.astype(np.int64), rec, n_k)
        for p in rng.uniform(0.01, 1.0, 5):
            out = C.c_int64()
            O._load_ref().ref_budget_for_recovery(pts.size, n_k, np.ascontiguousarray(pts, np.int64),
                                                  np.ascontiguousarray(rec), float(p), C.byref(out))
            assert c.budget_for_recovery(float(p)) == out.value
