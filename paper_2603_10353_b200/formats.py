"""Version-1 file formats of the reference CLI, so the GPU
runner consumes budget tables, head plans and recovery profiles written by the
reference with zero translation, and writes files the reference loads.

* allocation.json  save_allocation / load_allocation (proj/src/allocator.cpp:223-275)
* assignment.json  save_assignment / load_assignment (proj/src/partitioner.cpp:268-336)
* profiles.json    save_profiles / load_profiles     (proj/src/profiler.cpp:300-383)

Loaders are as strict as the reference's (json_util.hpp: unknown fields,
missing fields, wrong types, version != 1 are errors) and raise
``ShplbRuntimeError`` (a RuntimeError) with the reference's message text where
the reference throws std::runtime_error, ``InvalidArgument`` where it throws
std::invalid_argument. Writers reproduce the reference's byte layout
(nlohmann ``dump(2)``: sorted keys, two-space indent, arrays of numbers inline).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

from ._native import InvalidArgument, ShplbRuntimeError
from .api import RecoveryCurve


# --------------------------------------------------------------------------
# json_util.hpp helpers
# --------------------------------------------------------------------------

def _parse_file(path: str):
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ShplbRuntimeError(f"cannot open {path}") from None
    try:
        return json.loads(text)
    except json.JSONDecodeError as e:
        raise ShplbRuntimeError(f"{path}: {e}") from None


def _is_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _is_number(v) -> bool:
    return (isinstance(v, (int, float))) and not isinstance(v, bool)


def _expect_keys(j, where: str, allowed) -> None:
    if not isinstance(j, dict):
        raise ShplbRuntimeError(f"{where}: expected an object")
    for key in j:
        if key not in allowed:
            raise ShplbRuntimeError(f'{where}: unknown field "{key}"')


def _require(j, where: str, key: str):
    if key not in j:
        raise ShplbRuntimeError(f'{where}: missing field "{key}"')
    return j[key]


def _require_int(j, where: str, key: str) -> int:
    v = _require(j, where, key)
    if not _is_int(v):
        raise ShplbRuntimeError(f"{where}.{key}: expected an integer")
    return int(v)


def _require_number(j, where: str, key: str) -> float:
    v = _require(j, where, key)
    if not _is_number(v):
        raise ShplbRuntimeError(f"{where}.{key}: expected a number")
    return float(v)


def _require_string(j, where: str, key: str) -> str:
    v = _require(j, where, key)
    if not isinstance(v, str):
        raise ShplbRuntimeError(f"{where}.{key}: expected a string")
    return v


def _require_version_1(j, where: str) -> None:
    if _require_int(j, where, "version") != 1:
        raise ShplbRuntimeError(f"{where}: unsupported version (expected 1)")


def _num(v) -> str:
    if isinstance(v, float):
        if math.isnan(v) or math.isinf(v):
            return "null"  # nlohmann writes non-finite numbers as null
        r = repr(v)
        return r if ("." in r or "e" in r or "n" in r) else r + ".0"
    return str(int(v))


def _dump(v, indent: int = 0) -> str:
    """nlohmann::json::dump(2) layout: objects one key per line, sorted keys;
    arrays whose elements are all primitives inline without spaces."""
    pad = " " * indent
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f'{pad}  {json.dumps(k)}: {_dump(v[k], indent + 2)}' for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        if all(not isinstance(x, (dict, list, tuple)) for x in v):
            return "[" + ",".join(_dump(x) for x in v) + "]"
        items = [pad + "  " + _dump(x, indent + 2) for x in v]
        return "[\n" + ",\n".join(items) + "\n" + pad + "]"
    if isinstance(v, str):
        return json.dumps(v)
    if isinstance(v, bool):
        return "true" if v else "false"
    return _num(v)


def _write_file(path: str, obj) -> None:
    try:
        with open(path, "w") as f:
            f.write(_dump(obj) + "\n")
    except OSError:
        raise ShplbRuntimeError(f"cannot write {path}") from None


def _head_ids(heads, n):
    if heads is None:
        return [(0, h) for h in range(n)]
    heads = [(int(a), int(b)) for a, b in heads]
    if len(heads) != n:
        raise InvalidArgument("head identity list does not match the assignment")
    return heads


# --------------------------------------------------------------------------
# allocation.json (allocator.cpp:223-275)
# --------------------------------------------------------------------------

@dataclass
class LoadedAllocation:
    budgets: np.ndarray              # int64 [heads], tokens
    heads: list = field(default_factory=list)  # [(layer, head)]
    total: int = 0
    floor: int = 0


def save_allocation(path: str, budgets, total: int, floor: int, heads=None) -> None:
    """save_allocation (allocator.cpp:223-238)."""
    budgets = [int(b) for b in np.asarray(budgets, np.int64).ravel()]
    if not budgets or (heads is not None and len(heads) != len(budgets)):
        raise InvalidArgument("allocation must pair every head with a budget")
    ids = _head_ids(heads, len(budgets))
    _write_file(path, {"version": 1, "total": int(total), "floor": int(floor),
                       "budgets": [{"layer": l, "head": h, "budget": b} for (l, h), b in zip(ids, budgets)]})


def load_allocation(path: str) -> LoadedAllocation:
    """load_allocation (allocator.cpp:240-273): strict schema, every budget >=
    floor, budgets must sum to total."""
    j = _parse_file(path)
    _expect_keys(j, path, {"version", "total", "floor", "budgets"})
    _require_version_1(j, path)
    total = _require_int(j, path, "total")
    floor = _require_int(j, path, "floor")
    arr = _require(j, path, "budgets")
    if not isinstance(arr, list) or not arr:
        raise ShplbRuntimeError(f"{path}.budgets: expected a nonempty array")
    heads, budgets, s = [], [], 0
    for i, e in enumerate(arr):
        where = f"{path}.budgets[{i}]"
        _expect_keys(e, where, {"layer", "head", "budget"})
        layer = _require_int(e, where, "layer")
        head = _require_int(e, where, "head")
        b = _require_int(e, where, "budget")
        if b < floor:
            raise ShplbRuntimeError(f"{where}: budget {b} below the floor {floor}")
        heads.append((layer, head))
        budgets.append(b)
        s += b
    if s != total:
        raise ShplbRuntimeError(f"{path}: budgets sum to {s} but total says {total}")
    return LoadedAllocation(np.asarray(budgets, np.int64), heads, total, floor)


# --------------------------------------------------------------------------
# assignment.json (partitioner.cpp:268-336)
# --------------------------------------------------------------------------

@dataclass
class LoadedAssignment:
    device_of_head: np.ndarray       # int32 [heads]
    heads: list                      # [(layer, head)]
    devices: int
    loads: np.ndarray                # int64 [devices]
    total: int
    imbalance: float


def _validate_assignment(device_of_head, devices) -> None:
    # Assignment::validate (partitioner.cpp:38-48)
    if devices < 1:
        raise InvalidArgument("need at least one device")
    if len(device_of_head) == 0:
        raise InvalidArgument("assignment covers no heads")
    for h, d in enumerate(device_of_head):
        if d < 0 or d >= devices:
            raise InvalidArgument(f"head {h} assigned to invalid device {int(d)}")


def save_assignment(path: str, device_of_head, devices: int, loads, imbalance: float, heads=None) -> None:
    """save_assignment (partitioner.cpp:268-286); loads / imbalance as
    imbalance() reports them (api.imbalance)."""
    dev = [int(d) for d in np.asarray(device_of_head).ravel()]
    _validate_assignment(dev, devices)
    ids = _head_ids(heads, len(dev))
    _write_file(path, {"version": 1, "devices": int(devices),
                       "assignment": [{"layer": l, "head": h, "device": d} for (l, h), d in zip(ids, dev)],
                       "loads": [int(x) for x in np.asarray(loads).ravel()], "imbalance": float(imbalance)})


def load_assignment(path: str) -> LoadedAssignment:
    """load_assignment (partitioner.cpp:288-334)."""
    j = _parse_file(path)
    _expect_keys(j, path, {"version", "devices", "assignment", "loads", "imbalance"})
    _require_version_1(j, path)
    devices = _require_int(j, path, "devices")
    arr = _require(j, path, "assignment")
    if not isinstance(arr, list) or not arr:
        raise ShplbRuntimeError(f"{path}.assignment: expected a nonempty array")
    seen, heads, dev = set(), [], []
    for i, e in enumerate(arr):
        where = f"{path}.assignment[{i}]"
        _expect_keys(e, where, {"layer", "head", "device"})
        hid = (_require_int(e, where, "layer"), _require_int(e, where, "head"))
        if hid in seen:
            raise ShplbRuntimeError(f"{where}: head assigned twice")
        seen.add(hid)
        heads.append(hid)
        dev.append(_require_int(e, where, "device"))
    try:
        _validate_assignment(dev, devices)
    except InvalidArgument as e:
        raise ShplbRuntimeError(f"{path}: {e}") from None
    loads = _require(j, path, "loads")
    if not isinstance(loads, list) or len(loads) != devices:
        raise ShplbRuntimeError(f"{path}.loads: expected one entry per device")
    for v in loads:
        if not _is_int(v):
            raise ShplbRuntimeError(f"{path}.loads: expected integers")
    imb = _require_number(j, path, "imbalance")
    if imb < 1.0 - 1e-12:
        raise ShplbRuntimeError(f"{path}.imbalance: must be >= 1")
    return LoadedAssignment(np.asarray(dev, np.int32), heads, devices, np.asarray(loads, np.int64),
                            int(sum(loads)), imb)


# --------------------------------------------------------------------------
# profiles.json (profiler.cpp:300-383)
# --------------------------------------------------------------------------

POLICIES = ("per_query_topk", "column_aggregate_topk")
_CURVE_SLACK = 1e-12
_ENDPOINT_TOL = 1e-9


@dataclass
class LoadedProfiles:
    curves: list                     # [RecoveryCurve]
    heads: list                      # [(layer, head)]
    policy: str
    context_length: int
    provenance: list                 # [(request, task)] per profile


def _validate_curve(budgets, recovery, n_k) -> None:
    # RecoveryCurve::validate (profiler.cpp:25-54)
    if len(budgets) == 0:
        raise InvalidArgument("curve has no points")
    if n_k < 1:
        raise InvalidArgument("curve context_length must be >= 1")
    for i, (b, r) in enumerate(zip(budgets, recovery)):
        if b < 0 or b > n_k:
            raise InvalidArgument(f"budget out of [0, n_k] at points[{i}]")
        if r < -_CURVE_SLACK or r > 1.0 + _CURVE_SLACK:
            raise InvalidArgument(f"recovery out of [0, 1] at points[{i}]")
        if i > 0:
            if b <= budgets[i - 1]:
                raise InvalidArgument("budgets not strictly increasing")
            if r < recovery[i - 1] - _CURVE_SLACK:
                raise InvalidArgument(f"recovery decreasing at points[{i}]")
    if budgets[-1] != n_k:
        raise InvalidArgument("final point must sample the full context (k = n_k)")
    if abs(recovery[-1] - 1.0) > _ENDPOINT_TOL:
        raise InvalidArgument("final recovery must be 1 within 1e-9")


def save_profiles(path: str, curves, heads=None, policy: str = "per_query_topk",
                  request: str = "calibration", task: str = "synthetic") -> None:
    """save_profiles (profiler.cpp:300-330). curves: [RecoveryCurve] sharing
    one context length; provenance (request, task) applies to every profile."""
    if not curves:
        raise InvalidArgument("no profiles to save")
    if policy not in POLICIES:
        raise InvalidArgument(f'unknown selection policy "{policy}" '
                              "(expected per_query_topk or column_aggregate_topk)")
    if not request or not task:
        raise InvalidArgument("provenance request is empty" if not request else "provenance task is empty")
    for c in curves:
        _validate_curve([int(b) for b in c.budgets], [float(r) for r in c.recovery], int(c.context_length))
    n_k = int(curves[0].context_length)
    if any(int(c.context_length) != n_k for c in curves):
        raise InvalidArgument("profiles in one file must share the policy and context length")
    ids = _head_ids(heads, len(curves))
    _write_file(path, {"version": 1, "policy": policy, "context_length": n_k,
                       "profiles": [{"layer": l, "head": h,
                                     "points": [[int(b), float(r)] for b, r in zip(c.budgets, c.recovery)],
                                     "provenance": {"request": request, "task": task}}
                                    for (l, h), c in zip(ids, curves)]})


def load_profiles(path: str) -> LoadedProfiles:
    """load_profiles (profiler.cpp:332-383)."""
    j = _parse_file(path)
    _expect_keys(j, path, {"version", "policy", "context_length", "profiles"})
    _require_version_1(j, path)
    policy = _require_string(j, path, "policy")
    if policy not in POLICIES:  # selection_kind_from_string throws invalid_argument (workload.cpp:12-17)
        raise InvalidArgument(f'unknown selection policy "{policy}" '
                              "(expected per_query_topk or column_aggregate_topk)")
    n_k = _require_int(j, path, "context_length")
    arr = _require(j, path, "profiles")
    if not isinstance(arr, list) or not arr:
        raise ShplbRuntimeError(f"{path}.profiles: expected a nonempty array")
    curves, heads, prov = [], [], []
    for i, p in enumerate(arr):
        where = f"{path}.profiles[{i}]"
        _expect_keys(p, where, {"layer", "head", "points", "provenance"})
        hid = (_require_int(p, where, "layer"), _require_int(p, where, "head"))
        points = _require(p, where, "points")
        if not isinstance(points, list):
            raise ShplbRuntimeError(f"{where}.points: expected an array")
        budgets, recovery = [], []
        for k, pt in enumerate(points):
            if not (isinstance(pt, list) and len(pt) == 2 and _is_int(pt[0]) and _is_number(pt[1])):
                raise ShplbRuntimeError(f"{where}.points[{k}]: expected [budget:int, recovery:number]")
            budgets.append(int(pt[0]))
            recovery.append(float(pt[1]))
        pv = _require(p, where, "provenance")
        _expect_keys(pv, where + ".provenance", {"request", "task"})
        req = _require_string(pv, where + ".provenance", "request")
        tsk = _require_string(pv, where + ".provenance", "task")
        try:  # HeadProfile::validate (profiler.cpp:74-78)
            _validate_curve(budgets, recovery, n_k)
            if not req:
                raise InvalidArgument("provenance request is empty")
            if not tsk:
                raise InvalidArgument("provenance task is empty")
        except InvalidArgument as e:
            raise ShplbRuntimeError(f"{where}: {e}") from None
        curves.append(RecoveryCurve(np.asarray(budgets, np.int64), np.asarray(recovery, np.float64), n_k))
        heads.append(hid)
        prov.append((req, tsk))
    return LoadedProfiles(curves, heads, policy, n_k, prov)


def _pearson(a, b) -> float:
    # pearson (profiler.cpp:212-229), same accumulation order
    n = float(len(a))
    mean_a = mean_b = 0.0
    for x, y in zip(a, b):
        mean_a += x
        mean_b += y
    mean_a /= n
    mean_b /= n
    cov = var_a = var_b = 0.0
    for x, y in zip(a, b):
        da, db = x - mean_a, y - mean_b
        cov += da * db
        var_a += da * da
        var_b += db * db
    return cov / math.sqrt(var_a * var_b)


def stability_score(request_groups, p: float, normalization: str = "max") -> float:
    """stability_score (profiler.hpp:98-104, profiler.cpp:233-292): the paper's
    cross-request stability of relative head sparsity. Each
    group is one calibration request's LoadedProfiles; per request the per-head
    budget_for_recovery(p) vector (heads in (layer, head) order) is normalised
    by its max ("max") or sum ("sum"), and the minimum pairwise Pearson
    correlation is returned. Same errors and messages as the reference."""
    if len(request_groups) < 2:
        raise InvalidArgument("stability_score needs at least 2 calibration requests")
    if normalization not in ("max", "sum"):
        raise InvalidArgument('normalization must be "max" or "sum"')
    vectors, id_sets = [], []
    for g, group in enumerate(request_groups):
        prov = getattr(group, "provenance", None) or []
        name = prov[0][0] if prov and prov[0][0] else f"request #{g}"
        if not group.curves:
            raise InvalidArgument(f"{name}: empty profile group")
        heads = group.heads or [(0, h) for h in range(len(group.curves))]
        order = sorted(range(len(group.curves)), key=lambda i: tuple(heads[i]))
        budgets, ids = [], []
        for i in order:
            c = group.curves[i]
            budgets.append(float(c.budget_for_recovery(p)))
            ids.append(tuple(heads[i]))
        if g > 0 and ids != id_sets[0]:
            raise InvalidArgument(f"{name}: head set differs from the first request")
        denom = max(budgets) if normalization == "max" else sum(budgets)  # std::accumulate order
        if denom <= 0.0:
            raise InvalidArgument(f"{name}: budget vector cannot be normalized")
        budgets = [b / denom for b in budgets]
        if all(b == budgets[0] for b in budgets):
            raise InvalidArgument(f"{name}: budget vector has zero variance, correlation undefined")
        vectors.append(budgets)
        id_sets.append(ids)
    worst = 1.0
    for i in range(len(vectors)):
        for j in range(i + 1, len(vectors)):
            worst = min(worst, _pearson(vectors[i], vectors[j]))
    return worst
