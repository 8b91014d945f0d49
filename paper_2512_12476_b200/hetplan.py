"""Python mirror of the reference planner's API over the engine's C ABI.

The reference ("hetplan", /root/reference/proj) is a C++20 library whose
hot path is ``nested_sha_search`` -> ``ga_run`` -> ``evaluate`` ->
``balance_data`` / ``balance_layers`` / ``end_to_end_cost``
(proj/src/search.cpp:259-279, 437-835; proj/src/cost_model.cpp:431-487).
This module exposes the same entry points with the same argument meaning,
backed by ``libhpg.so`` (include/hpg.h): CUDA kernels for sm_100a plus a
C++20 host. There is no CPU fallback: constructing an :class:`Engine`
without the built library or without a Blackwell GPU raises.

Plans are plain dicts mirroring ``hetplan::Plan`` (plan.hpp:59-70)::

    {"groups": [[1, 2], [3, 6]],          # TaskGrouping (task ids)
     "counts": [16, 16],                  # GpuGrouping
     "layouts": {1: {"dp":..,"pp":..,"tp":..,"stage_layers":[..],
                     "weights":[..]}},    # ParallelLayout per task id
     "assignment": {1: [device indices in flat (replica, stage, shard)
                        order]}}

Devices are topology indices (the reference keys them by id string; the
index <-> id map is the topology's device order, as in resolve_plan).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
# HPG_LIBRARY selects another build of the engine (diagnostics: the
# bounds-checked libhpg_checked.so, `make -C paper_2512_12476_b200/csrc checked`)
LIB_PATH = os.environ.get("HPG_LIBRARY") or os.path.join(_HERE, "libhpg.so")

HPG_OK, HPG_USAGE, HPG_INPUT, HPG_INFEASIBLE, HPG_INTERNAL = 0, 2, 3, 4, 5


class HpgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InputError(HpgError):
    """hetplan::InputError (errors.hpp:11-14), CLI exit code 3."""


class UsageError(HpgError):
    """hetplan::UsageError (errors.hpp:16-18), CLI exit code 2."""


class InfeasibleError(HpgError):
    """no feasible plan (cli.cpp:104-108), exit code 4."""


class InternalError(HpgError):
    """engine / CUDA failure, exit code 5."""


def _raise(code: int, err) -> None:
    if code == HPG_OK:
        return
    msg = err.value.decode(errors="replace") if hasattr(err, "value") else str(err)
    cls = {HPG_USAGE: UsageError, HPG_INPUT: InputError,
           HPG_INFEASIBLE: InfeasibleError}.get(code, InternalError)
    raise cls(code, msg)


# ---- ctypes mirrors of include/hpg.h ----

class _Device(C.Structure):
    _fields_ = [("id", C.c_char_p), ("gpu_model", C.c_char_p), ("comp_tflops", C.c_double),
                ("mem_gb", C.c_double), ("hbm_gbps", C.c_double),
                ("intra_node_gbps", C.c_double), ("node", C.c_char_p), ("region", C.c_char_p)]


class _RegionLink(C.Structure):
    _fields_ = [("src", C.c_char_p), ("dst", C.c_char_p), ("latency_ms", C.c_double),
                ("bandwidth_gbps", C.c_double)]


class _Task(C.Structure):
    _fields_ = [("id", C.c_int32), ("kind", C.c_int32), ("hidden_size", C.c_int64),
                ("intermediate_size", C.c_int64), ("num_layers", C.c_int64),
                ("include_embedding", C.c_int32), ("vocab_size", C.c_int64),
                ("precision_bytes", C.c_int32)]


class _Problem(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("mode", C.c_int32), ("eta", C.c_double),
                ("global_batch", C.c_int64), ("responses_per_prompt", C.c_int64),
                ("seq_in", C.c_int64), ("seq_out", C.c_int64), ("micro_batch_size", C.c_int64),
                ("n_tasks", C.c_int32), ("tasks", C.POINTER(_Task)),
                ("n_dep_edges", C.c_int32), ("dep_edges", C.POINTER(C.c_int32)),
                ("n_devices", C.c_int32), ("devices", C.POINTER(_Device)),
                ("n_region_links", C.c_int32), ("region_links", C.POINTER(_RegionLink)),
                ("intra_region_latency_ms", C.c_double),
                ("intra_region_bandwidth_gbps", C.c_double)]


class _CostConfig(C.Structure):
    _fields_ = [("recompute", C.c_int32), ("reshard_override", C.c_double),
                ("sync_override", C.c_double), ("dbs_override", C.c_double),
                ("train_bytes_per_param", C.c_double), ("infer_bytes_per_param", C.c_double),
                ("kv_bytes_per_elem", C.c_double), ("dbs_cap", C.c_int32),
                ("act_factor", C.c_double)]


class _PlanTable(C.Structure):
    _fields_ = [("n_plans", C.c_int32), ("n_groups", C.POINTER(C.c_int32)),
                ("task_group", C.POINTER(C.c_int32)), ("gpu_counts", C.POINTER(C.c_int32)),
                ("dp", C.POINTER(C.c_int32)), ("pp", C.POINTER(C.c_int32)),
                ("tp", C.POINTER(C.c_int32)), ("sl_off", C.POINTER(C.c_int64)),
                ("stage_layers", C.POINTER(C.c_int32)), ("w_off", C.POINTER(C.c_int64)),
                ("weights", C.POINTER(C.c_double)), ("dev_off", C.POINTER(C.c_int64)),
                ("devices", C.POINTER(C.c_int32))]


class _EvalOut(C.Structure):
    _fields_ = [("end_to_end_s", C.POINTER(C.c_double)),
                ("memory_feasible", C.POINTER(C.c_uint8)),
                ("per_task", C.POINTER(C.c_double)), ("reshard_s", C.POINTER(C.c_double)),
                ("sync_s", C.POINTER(C.c_double))]


class _Knobs(C.Structure):
    _fields_ = [("budget", C.c_int64), ("seed", C.c_uint64), ("population", C.c_int32),
                ("locality_bias", C.c_double), ("quantize_gpu_counts", C.c_int32),
                ("level1_filter_adjacent", C.c_int32), ("level1_cap", C.c_int32),
                ("gg_arm_cap", C.c_int32), ("swap_pair_sample", C.c_int32),
                ("balance_data", C.c_int32), ("balance_layers", C.c_int32),
                ("balance_seqlen", C.c_int32), ("recompute", C.c_int32),
                ("reshard_override", C.c_double), ("sync_override", C.c_double),
                ("n_tg_override", C.c_int32), ("tg_override", C.POINTER(C.c_int32)),
                ("exhaustive_cap", C.c_double)]


class _SearchInfo(C.Structure):
    _fields_ = [("budget", C.c_int64), ("consumed", C.c_int64), ("seed", C.c_uint64),
                ("has_plan", C.c_int32), ("n_b_m", C.c_int32), ("n_trace", C.c_int32),
                ("n_arms", C.c_int32), ("n_halvings", C.c_int32),
                ("n_survivor_sets", C.c_int32), ("task_groupings", C.c_int64),
                ("wall_s", C.c_double), ("time_to_best_s", C.c_double),
                ("gpu_launches", C.c_int64), ("waves", C.c_int64),
                ("plans_evaluated_gpu", C.c_int64), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("eval_kernel_ms", C.c_double),
                ("eval_launches", C.c_int64), ("canonical_bytes", C.c_int64),
                ("host_ms", C.c_double), ("batch_ms", C.c_double)]


class _ResolvedTask(C.Structure):
    _fields_ = [("task_slot", C.c_int32), ("dp", C.c_int32), ("pp", C.c_int32), ("tp", C.c_int32),
                ("stage_layers", C.POINTER(C.c_int32)), ("nm_replica", C.POINTER(C.c_int64)),
                ("devices", C.POINTER(C.c_int32))]


class _Improvement(C.Structure):
    _fields_ = [("run", C.c_int64), ("local_idx", C.c_int64), ("cost", C.c_double)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class _SweepStats(C.Structure):
    _fields_ = [("best_cost", C.c_double), ("best_k", C.c_uint64), ("n_feasible", C.c_uint64),
                ("xor_bits", C.c_uint64), ("canonical_bytes", C.c_uint64),
                ("total_ms", C.c_double), ("eval_ms", C.c_double), ("gen_ms", C.c_double),
                ("launches", C.c_int64), ("global_slab_plans", C.c_uint64)]


_lib = None

EXPORTED_SYMBOLS = [
    "hpg_abi_version", "hpg_cost_config_default", "hpg_knobs_default", "hpg_create",
    "hpg_destroy", "hpg_restage", "hpg_max_devices_per_node", "hpg_link", "hpg_eval", "hpg_check_memory",
    "hpg_balance", "hpg_search", "hpg_nccl_unique_id", "hpg_search_dist", "hpg_ga_search",
    "hpg_result_info", "hpg_result_b_m", "hpg_result_trace", "hpg_result_arms",
    "hpg_result_halvings", "hpg_result_survivor_sizes", "hpg_result_survivors",
    "hpg_result_plan", "hpg_result_breakdown", "hpg_result_free", "hpg_sweep",
    "hpg_sweep_resident", "hpg_sweep_dist", "hpg_exhaustive", "hpg_exhaustive_estimate",
    "hpg_task_cost", "hpg_ring_bottleneck", "hpg_pair_cost", "hpg_dist_exchange",
]


def load_library(path: str = LIB_PATH):
    """Loads libhpg.so (raises if it was not built: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run __graft_entry__.build() (no CPU fallback)")
    lib = C.CDLL(path)
    P = C.POINTER
    E = C.c_char_p
    L = C.c_size_t
    sig = {
        "hpg_abi_version": (C.c_int, []),
        "hpg_cost_config_default": (None, [P(_CostConfig)]),
        "hpg_knobs_default": (None, [P(_Knobs)]),
        "hpg_create": (C.c_int, [P(_Problem), C.c_int, P(C.c_void_p), E, L]),
        "hpg_destroy": (None, [C.c_void_p]),
        "hpg_restage": (C.c_int, [C.c_void_p, P(_Problem), E, L]),
        "hpg_max_devices_per_node": (C.c_int, [C.c_void_p]),
        "hpg_link": (C.c_int, [C.c_void_p, C.c_int, C.c_int, P(C.c_double), P(C.c_double)]),
        "hpg_eval": (C.c_int, [C.c_void_p, P(_PlanTable), P(_CostConfig), P(_EvalOut), E, L]),
        "hpg_check_memory": (C.c_int, [C.c_void_p, P(_PlanTable), P(_CostConfig),
                                       P(C.c_uint8), P(C.c_double), E, L]),
        "hpg_balance": (C.c_int, [C.c_void_p, P(_PlanTable), P(_CostConfig), C.c_int,
                                  P(C.c_int32), P(C.c_double), P(C.c_double), E, L]),
        "hpg_search": (C.c_int, [C.c_void_p, P(_Knobs), P(C.c_void_p), E, L]),
        "hpg_nccl_unique_id": (C.c_int, [P(C.c_uint8), E, L]),
        "hpg_search_dist": (C.c_int, [C.c_void_p, P(_Knobs), C.c_int, C.c_int, P(C.c_uint8),
                                      P(C.c_void_p), E, L]),
        "hpg_ga_search": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_int32, P(C.c_int32),
                                    C.c_int64, C.c_uint64, P(_Knobs), P(C.c_void_p), E, L]),
        "hpg_exhaustive": (C.c_int, [C.c_void_p, P(_Knobs), P(C.c_void_p), E, L]),
        "hpg_exhaustive_estimate": (C.c_int, [C.c_void_p, P(_Knobs), P(C.c_double), E, L]),
        "hpg_result_info": (C.c_int, [C.c_void_p, P(_SearchInfo)]),
        "hpg_result_b_m": (C.c_int, [C.c_void_p, P(C.c_int64)]),
        "hpg_result_trace": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_double)]),
        "hpg_result_arms": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_double),
                                      P(C.c_int64)]),
        "hpg_result_halvings": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_int64),
                                          P(C.c_int64), P(C.c_double), P(C.c_double)]),
        "hpg_result_survivor_sizes": (C.c_int, [C.c_void_p, P(C.c_int32)]),
        "hpg_result_survivors": (C.c_int, [C.c_void_p, P(C.c_int64)]),
        "hpg_result_plan": (C.c_int, [C.c_void_p, P(_PlanTable), P(C.c_int32), P(C.c_double),
                                      P(C.c_uint64), P(C.c_int64)]),
        "hpg_result_breakdown": (C.c_int, [C.c_void_p, P(C.c_double), P(C.c_double),
                                           P(C.c_double), P(C.c_double), P(C.c_uint8)]),
        "hpg_result_free": (None, [C.c_void_p]),
        "hpg_sweep": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, P(C.c_double),
                                P(C.c_uint8), P(C.c_double), P(C.c_uint64), P(C.c_uint64), E, L]),
        "hpg_sweep_resident": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                         P(_SweepStats), E, L]),
        "hpg_sweep_dist": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                     P(C.c_uint8), P(_SweepStats), E, L]),
        "hpg_task_cost": (C.c_int, [C.c_void_p, P(_ResolvedTask), P(_CostConfig), P(C.c_double),
                                    P(C.c_double), P(C.c_double), P(C.c_double), E, L]),
        "hpg_ring_bottleneck": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_int32, C.c_double,
                                          P(C.c_double), E, L]),
        "hpg_pair_cost": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_int32, P(C.c_int32), C.c_int32,
                                    C.c_double, P(C.c_double), E, L]),
        "hpg_dist_exchange": (C.c_int, [C.c_int, C.c_int, ALLGATHER_FN, C.c_void_p, C.c_int32,
                                        P(C.c_int64), P(C.c_int32), P(C.c_int64), P(C.c_double),
                                        P(_Improvement), C.c_int64, P(_Improvement), C.c_int64,
                                        P(C.c_int64), E, L]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


# ---- input parsing (reference JSON formats + the oracle's hex-float dumps) ----

def _f(v) -> float:
    if isinstance(v, str):
        return float.fromhex(v)
    return float(v)


TASK_KIND = {1: 0, 2: 1, 3: 1, 4: 1, 5: 2, 6: 2}   # workflow.cpp:85-93
TASK_MODEL = {1: "actor", 2: "reward", 3: "reference", 4: "critic", 5: "critic", 6: "actor"}


@dataclass
class Workflow:
    """hetplan::WorkflowGraph (workflow.hpp:67-77)."""
    algorithm: str = "ppo"
    mode: str = "sync"
    eta: float = 0.5
    global_batch: int = 1
    responses_per_prompt: int = 1
    seq_in: int = 1
    seq_out: int = 0
    micro_batch_size: int = 1
    tasks: List[dict] = field(default_factory=list)   # id, kind, h1, h2, nl, emb, vocab, prec
    dep_edges: List[tuple] = field(default_factory=list)

    @property
    def task_ids(self) -> List[int]:
        return [t["id"] for t in self.tasks]


def build_workflow(algorithm: str, mode: str, models: Dict[str, dict], batch: dict,
                   eta: float) -> Workflow:
    """build_workflow (workflow.cpp:97-146)."""
    ids = [1, 2, 3, 4, 5, 6] if algorithm == "ppo" else [1, 2, 3, 6]
    wf = Workflow(algorithm=algorithm, mode=mode, eta=eta,
                  global_batch=batch["global_batch"],
                  responses_per_prompt=batch["responses_per_prompt"],
                  seq_in=batch["seq_in"], seq_out=batch["seq_out"],
                  micro_batch_size=batch["micro_batch_size"])
    for i in ids:
        name = TASK_MODEL[i]
        if name not in models:
            raise InputError(HPG_INPUT, f"missing model spec '{name}' required by task {i}")
        m = models[name]
        wf.tasks.append(dict(id=i, kind=TASK_KIND[i], h1=m["hidden_size"],
                             h2=m["intermediate_size"], nl=m["num_layers"],
                             emb=bool(m.get("include_embedding", False)),
                             vocab=m.get("vocab_size", 0), prec=2,
                             model_name=name))
    infs = [t["id"] for t in wf.tasks if t["kind"] == 1]
    trs = [t["id"] for t in wf.tasks if t["kind"] == 2]
    edges = set((1, i) for i in infs) | set((i, t) for i in infs for t in trs)
    wf.dep_edges = sorted(edges)
    return wf


def parse_workflow(obj: dict) -> Workflow:
    """Reference workflow JSON (parse_workflow_json, workflow.cpp:177-232) or the
    oracle's explicit-task dump."""
    if "tasks" in obj:
        wf = Workflow(algorithm=obj["algorithm"], mode=obj["mode"], eta=_f(obj["eta"]),
                      global_batch=obj["batch"]["global_batch"],
                      responses_per_prompt=obj["batch"]["responses_per_prompt"],
                      seq_in=obj["batch"]["seq_in"], seq_out=obj["batch"]["seq_out"],
                      micro_batch_size=obj["batch"]["micro_batch_size"])
        for t in obj["tasks"]:
            wf.tasks.append(dict(id=t["id"], kind=t["kind"], h1=t["hidden_size"],
                                 h2=t["intermediate_size"], nl=t["num_layers"],
                                 emb=bool(t["include_embedding"]), vocab=t["vocab_size"],
                                 prec=t["precision_bytes"], model_name=t.get("model_name", "")))
        wf.dep_edges = [tuple(e) for e in obj.get("dep_edges", [])]
        return wf
    wf = build_workflow(obj["algorithm"], obj["mode"], obj["models"], obj["batch"],
                        _f(obj.get("eta", 0.5)))
    for name, prec in obj.get("precision_bytes", {}).items():
        for t in wf.tasks:
            if t["model_name"] == name:
                t["prec"] = int(prec)
    return wf


@dataclass
class Topology:
    """DeviceTopology inputs (topology.hpp:59-104)."""
    devices: List[dict]
    region_links: List[dict]
    defaults: dict

    @property
    def n(self) -> int:
        return len(self.devices)

    def device_index(self, dev_id: str) -> int:
        for i, d in enumerate(self.devices):
            if d["id"] == dev_id:
                return i
        raise InputError(HPG_INPUT, f"unknown device id '{dev_id}'")


def parse_topology(obj: dict) -> Topology:
    devs = [dict(id=d["id"], gpu_model=d["gpu_model"], comp_tflops=_f(d["comp_tflops"]),
                 mem_gb=_f(d["mem_gb"]), hbm_gbps=_f(d["hbm_gbps"]),
                 intra_node_gbps=_f(d["intra_node_gbps"]), node=d["node"], region=d["region"])
            for d in obj["devices"]]
    links = [dict(src=l["src"], dst=l["dst"], latency_ms=_f(l["latency_ms"]),
                  bandwidth_gbps=_f(l["bandwidth_gbps"])) for l in obj.get("region_links", [])]
    d = obj.get("defaults", {})
    defaults = dict(intra_region_latency_ms=_f(d.get("intra_region_latency_ms", 0.1)),
                    intra_region_bandwidth_gbps=_f(d.get("intra_region_bandwidth_gbps", 100.0)))
    return Topology(devs, links, defaults)


def load_workflow(path: str) -> Workflow:
    with open(path) as f:
        return parse_workflow(json.load(f))


def load_topology(path: str) -> Topology:
    with open(path) as f:
        return parse_topology(json.load(f))


@dataclass
class CostModelConfig:
    """CostModelConfig + MemoryModel (cost_model.hpp:13-28, plan.hpp:83-89)."""
    recompute: bool = True
    reshard_override: float = -1.0
    sync_override: float = -1.0
    dbs_override: float = -1.0
    train_bytes_per_param: float = 18.0
    infer_bytes_per_param: float = 2.0
    kv_bytes_per_elem: float = 2.0
    dbs_cap: int = 1
    act_factor: float = 4.0

    @staticmethod
    def from_json(obj: dict) -> "CostModelConfig":
        m = obj.get("memory", {})
        return CostModelConfig(
            recompute=bool(obj.get("recompute", True)),
            reshard_override=_f(obj.get("reshard_override", -1.0)),
            sync_override=_f(obj.get("sync_override", -1.0)),
            dbs_override=_f(obj.get("dbs_override", -1.0)),
            train_bytes_per_param=_f(m.get("train_bytes_per_param", 18.0)),
            infer_bytes_per_param=_f(m.get("infer_bytes_per_param", 2.0)),
            kv_bytes_per_elem=_f(m.get("kv_bytes_per_elem", 2.0)),
            dbs_cap=int(m.get("dbs_cap", 1)), act_factor=_f(m.get("act_factor", 4.0)))

    def _c(self) -> _CostConfig:
        return _CostConfig(int(self.recompute), self.reshard_override, self.sync_override,
                           self.dbs_override, self.train_bytes_per_param,
                           self.infer_bytes_per_param, self.kv_bytes_per_elem, self.dbs_cap,
                           self.act_factor)


@dataclass
class SearchKnobs:
    """SearchKnobs (search.hpp:17-39); defaults = the reference defaults."""
    budget: int = 1000
    seed: int = 0
    population: int = 16
    locality_bias: float = 0.8
    quantize_gpu_counts: int = 1
    level1_filter: str = "off"
    level1_cap: int = 0
    gg_arm_cap: int = 64
    swap_pair_sample: int = 8
    balance_data: bool = True
    balance_layers: bool = True
    balance_seqlen: bool = True
    recompute: bool = True
    reshard_override: float = -1.0
    sync_override: float = -1.0
    exhaustive_cap: float = 1e6

    @staticmethod
    def from_json(obj: dict) -> "SearchKnobs":
        k = SearchKnobs()
        for f_ in k.__dataclass_fields__:
            if f_ in obj:
                v = obj[f_]
                cur = getattr(k, f_)
                if isinstance(cur, bool):
                    v = bool(v)
                elif isinstance(cur, float):
                    v = _f(v)
                elif isinstance(cur, int):
                    v = int(v)
                setattr(k, f_, v)
        return k


# ---- plan tables ----

def _arr(ctype, values):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)


class PlanTable:
    """Struct-of-arrays hpg_plan_table built from plan dicts."""

    def __init__(self, plans: Sequence[dict], wf: Workflow):
        ids = wf.task_ids
        T = len(ids)
        n_groups, task_group, counts = [], [], []
        dp, pp, tp, sl_off, w_off, dev_off = [], [], [], [], [], []
        sls, ws, devs = [], [], []
        for p in plans:
            groups = p["groups"]
            n_groups.append(len(groups))
            g_of = {}
            for gi, g in enumerate(groups):
                for tid in g:
                    g_of[int(tid)] = gi
            for tid in ids:
                task_group.append(g_of.get(tid, -1))
            cc = list(p["counts"]) + [0] * (T - len(p["counts"]))
            counts.extend(cc[:T])
            lay = {int(k): v for k, v in p["layouts"].items()}
            asg = {int(k): v for k, v in p["assignment"].items()}
            for tid in ids:
                l = lay[tid]
                dp.append(l["dp"])
                pp.append(l["pp"])
                tp.append(l["tp"])
                sl_off.append(len(sls))
                sls.extend(l["stage_layers"])
                w_off.append(len(ws))
                w = l.get("weights", l.get("replica_batch_weights", [1.0] * l["dp"]))
                ws.extend(_f(x) for x in w)
                dev_off.append(len(devs))
                devs.extend(asg[tid])
        self._keep = [_arr(C.c_int32, n_groups), _arr(C.c_int32, task_group),
                      _arr(C.c_int32, counts), _arr(C.c_int32, dp), _arr(C.c_int32, pp),
                      _arr(C.c_int32, tp), _arr(C.c_int64, sl_off), _arr(C.c_int32, sls),
                      _arr(C.c_int64, w_off), _arr(C.c_double, ws), _arr(C.c_int64, dev_off),
                      _arr(C.c_int32, devs)]
        k = self._keep
        self.c = _PlanTable(len(plans), k[0], k[1], k[2], k[3], k[4], k[5], k[6], k[7], k[8],
                            k[9], k[10], k[11])
        self.n = len(plans)
        self.sl_off, self.w_off = sl_off, w_off
        self.n_sl, self.n_w = len(sls), len(ws)


COMPONENTS = ("comp", "tp", "pp", "dp", "bubble", "hbm", "total")


class Engine:
    """One problem (workflow + topology) staged on one GPU; hetplan's hot-path
    API as methods. Not thread-safe (like an hpg_ctx)."""

    def __init__(self, wf: Workflow, topo: Topology, device: int = 0):
        self.lib = load_library()
        prob = self._problem(wf, topo)
        self._h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = self.lib.hpg_create(C.byref(prob), device, C.byref(self._h), err, 1024)
        _raise(rc, err)

    def _problem(self, wf: Workflow, topo: Topology) -> "_Problem":
        """hpg_problem from host objects (kept alive on self)"""
        self.wf, self.topo = wf, topo
        tasks = (_Task * len(wf.tasks))(*[
            _Task(t["id"], t["kind"], t["h1"], t["h2"], t["nl"], int(t["emb"]), t["vocab"],
                  t["prec"]) for t in wf.tasks])
        edges = [x for e in wf.dep_edges for x in e]
        self._strings = []

        def s(x):
            b = x.encode()
            self._strings.append(b)
            return b
        devs = (_Device * topo.n)(*[
            _Device(s(d["id"]), s(d["gpu_model"]), d["comp_tflops"], d["mem_gb"],
                    d["hbm_gbps"], d["intra_node_gbps"], s(d["node"]), s(d["region"]))
            for d in topo.devices])
        links = (_RegionLink * max(1, len(topo.region_links)))(*[
            _RegionLink(s(l["src"]), s(l["dst"]), l["latency_ms"], l["bandwidth_gbps"])
            for l in topo.region_links])
        self._keep = (tasks, devs, links, _arr(C.c_int32, edges))
        return _Problem(0 if wf.algorithm == "ppo" else 1, 0 if wf.mode == "sync" else 1,
                        wf.eta, wf.global_batch, wf.responses_per_prompt, wf.seq_in,
                        wf.seq_out, wf.micro_batch_size, len(wf.tasks), tasks,
                        len(wf.dep_edges), self._keep[3], topo.n, devs,
                        len(topo.region_links), links,
                        topo.defaults["intra_region_latency_ms"],
                        topo.defaults["intra_region_bandwidth_gbps"])

    def restage(self, wf: Workflow, topo: Topology) -> None:
        """hpg_restage: upload a (new) problem into this context"""
        prob = self._problem(wf, topo)
        err = C.create_string_buffer(1024)
        _raise(self.lib.hpg_restage(self._h, C.byref(prob), err, 1024), err)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.hpg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def max_devices_per_node(self) -> int:
        return self.lib.hpg_max_devices_per_node(self._h)

    def link(self, a: int, b: int):
        lat, bw = C.c_double(), C.c_double()
        rc = self.lib.hpg_link(self._h, a, b, C.byref(lat), C.byref(bw))
        _raise(rc, "link index out of range")
        return lat.value, bw.value

    # ---- cost model (cost_model.hpp:103-117, plan.hpp:116-119) ----

    def end_to_end_cost(self, plans: Sequence[dict], cfg: Optional[CostModelConfig] = None,
                        per_task: bool = True) -> List[dict]:
        cfg = cfg or CostModelConfig()
        pt = PlanTable(plans, self.wf)
        n, T = pt.n, len(self.wf.tasks)
        e2e = (C.c_double * max(1, n))()
        feas = (C.c_uint8 * max(1, n))()
        rs = (C.c_double * max(1, n))()
        sy = (C.c_double * max(1, n))()
        ptk = (C.c_double * max(1, n * T * 7))() if per_task else None
        out = _EvalOut(e2e, feas, ptk, rs, sy)
        err = C.create_string_buffer(1024)
        c = cfg._c()
        rc = self.lib.hpg_eval(self._h, C.byref(pt.c), C.byref(c), C.byref(out), err, 1024)
        _raise(rc, err)
        res = []
        for i in range(n):
            bd = dict(end_to_end_s=e2e[i], memory_feasible=bool(feas[i]), reshard_s=rs[i],
                      sync_s=sy[i])
            if per_task:
                bd["per_task"] = {
                    self.wf.tasks[t]["id"]: {COMPONENTS[c_]: ptk[(i * T + t) * 7 + c_]
                                             for c_ in range(7)} for t in range(T)}
            res.append(bd)
        return res

    def check_memory(self, plans: Sequence[dict], cfg: Optional[CostModelConfig] = None):
        """Returns (feasible list, required bytes per plan per device)."""
        cfg = cfg or CostModelConfig()
        pt = PlanTable(plans, self.wf)
        n, N = pt.n, self.topo.n
        feas = (C.c_uint8 * max(1, n))()
        req = (C.c_double * max(1, n * N))()
        err = C.create_string_buffer(1024)
        c = cfg._c()
        rc = self.lib.hpg_check_memory(self._h, C.byref(pt.c), C.byref(c), feas, req, err, 1024)
        _raise(rc, err)
        return [bool(feas[i]) for i in range(n)], [[req[i * N + d] for d in range(N)]
                                                    for i in range(n)]

    def _balance(self, plans, cfg, which):
        cfg = cfg or CostModelConfig()
        pt = PlanTable(plans, self.wf)
        sl = (C.c_int32 * max(1, pt.n_sl))()
        w = (C.c_double * max(1, pt.n_w))()
        e2e = (C.c_double * max(1, pt.n))()
        err = C.create_string_buffer(1024)
        c = cfg._c()
        rc = self.lib.hpg_balance(self._h, C.byref(pt.c), C.byref(c), which, sl, w, e2e, err,
                                  1024)
        _raise(rc, err)
        out = []
        T = len(self.wf.tasks)
        for i, p in enumerate(plans):
            q = json.loads(json.dumps(p))
            q["layouts"] = {int(k): v for k, v in q["layouts"].items()}
            q["assignment"] = {int(k): v for k, v in q["assignment"].items()}
            for t, tid in enumerate(self.wf.task_ids):
                l = dict(q["layouts"][tid])
                so, wo = pt.sl_off[i * T + t], pt.w_off[i * T + t]
                l["stage_layers"] = [sl[so + j] for j in range(l["pp"])]
                l["weights"] = [w[wo + j] for j in range(l["dp"])]
                q["layouts"][tid] = l
            q["_e2e"] = e2e[i]
            out.append(q)
        return out

    def balance_data(self, plans, cfg=None):
        """balance_data (balance.cpp:37-56) per plan."""
        return self._balance(plans, cfg, 1)

    def balance_layers(self, plans, cfg=None):
        """balance_layers (balance.cpp:81-167) per plan."""
        return self._balance(plans, cfg, 2)

    def evaluate(self, plans, cfg=None):
        """EvalContext::evaluate's chain (search.cpp:259-279) per plan."""
        return self._balance(plans, cfg, 3)

    # ---- search (search.hpp:115-135) ----

    def _knobs(self, k: SearchKnobs, tg_override=None):
        kn = _Knobs()
        self.lib.hpg_knobs_default(C.byref(kn))
        kn.budget, kn.seed, kn.population = k.budget, k.seed, k.population
        kn.locality_bias, kn.quantize_gpu_counts = k.locality_bias, k.quantize_gpu_counts
        kn.level1_filter_adjacent = 1 if k.level1_filter == "adjacent" else 0
        kn.level1_cap, kn.gg_arm_cap, kn.swap_pair_sample = (k.level1_cap, k.gg_arm_cap,
                                                             k.swap_pair_sample)
        kn.balance_data, kn.balance_layers = int(k.balance_data), int(k.balance_layers)
        kn.balance_seqlen, kn.recompute = int(k.balance_seqlen), int(k.recompute)
        kn.reshard_override, kn.sync_override = k.reshard_override, k.sync_override
        kn.exhaustive_cap = k.exhaustive_cap
        keep = None
        if tg_override:
            ids = self.wf.task_ids
            flat = []
            for tg in tg_override:
                g_of = {tid: gi for gi, g in enumerate(tg) for tid in g}
                flat.extend(g_of[t] for t in ids)
            keep = _arr(C.c_int32, flat)
            kn.n_tg_override = len(tg_override)
            kn.tg_override = keep
        return kn, keep

    def nested_sha_search(self, knobs: SearchKnobs, tg_override=None) -> "SearchResult":
        kn, keep = self._knobs(knobs, tg_override)
        r = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = self.lib.hpg_search(self._h, C.byref(kn), C.byref(r), err, 1024)
        _raise(rc, err)
        return SearchResult(self, r)

    def nested_sha_search_dist(self, knobs: SearchKnobs, rank: int, world: int,
                               nccl_id: bytes) -> "SearchResult":
        kn, keep = self._knobs(knobs)
        r = C.c_void_p()
        err = C.create_string_buffer(1024)
        idb = (C.c_uint8 * 128)(*nccl_id)
        rc = self.lib.hpg_search_dist(self._h, C.byref(kn), rank, world, idb, C.byref(r), err,
                                      1024)
        _raise(rc, err)
        return SearchResult(self, r)

    def nccl_unique_id(self) -> bytes:
        buf = (C.c_uint8 * 128)()
        err = C.create_string_buffer(1024)
        _raise(self.lib.hpg_nccl_unique_id(buf, err, 1024), err)
        return bytes(buf)

    def ga_search(self, groups: List[List[int]], counts: List[int], budget_slice: int,
                  rng_seed: int, knobs: SearchKnobs) -> "SearchResult":
        kn, keep = self._knobs(knobs)
        g_of = {tid: gi for gi, g in enumerate(groups) for tid in g}
        tg = _arr(C.c_int32, [g_of[t] for t in self.wf.task_ids])
        cnt = _arr(C.c_int32, counts)
        r = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = self.lib.hpg_ga_search(self._h, tg, len(groups), cnt, budget_slice, rng_seed,
                                    C.byref(kn), C.byref(r), err, 1024)
        _raise(rc, err)
        return SearchResult(self, r)

    # ---- exhaustive oracle (search.hpp:137-155) ----

    def exhaustive_search(self, knobs: SearchKnobs) -> "SearchResult":
        """exhaustive_search on the device; result.info["consumed"] = explored
        (unique plans evaluated), result.info["budget"] = raw candidates."""
        kn, keep = self._knobs(knobs)
        r = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = self.lib.hpg_exhaustive(self._h, C.byref(kn), C.byref(r), err, 1024)
        _raise(rc, err)
        return SearchResult(self, r)

    def exhaustive_space_estimate(self, knobs: SearchKnobs) -> float:
        kn, keep = self._knobs(knobs)
        est = C.c_double()
        err = C.create_string_buffer(1024)
        _raise(self.lib.hpg_exhaustive_estimate(self._h, C.byref(kn), C.byref(est), err, 1024),
               err)
        return est.value

    # ---- config-5 sweep ----

    def sweep(self, seed: int, k0: int, count: int, want_costs: bool = True):
        costs = (C.c_double * max(1, count))() if want_costs else None
        feas = (C.c_uint8 * max(1, count))() if want_costs else None
        best, bk, nf = C.c_double(), C.c_uint64(), C.c_uint64()
        err = C.create_string_buffer(1024)
        rc = self.lib.hpg_sweep(self._h, seed, k0, count, costs, feas, C.byref(best),
                                C.byref(bk), C.byref(nf), err, 1024)
        _raise(rc, err)
        out = dict(best_cost=best.value, best_k=bk.value, n_feasible=nf.value)
        if want_costs:
            out["costs"] = [costs[i] for i in range(count)]
            out["feasible"] = [bool(feas[i]) for i in range(count)]
        return out

    # ---- cost-model primitives (cost_model.hpp:49-111) ----

    def task_cost_detail(self, task_slot: int, dp: int, pp: int, tp: int,
                         stage_layers: Sequence[int], nm_replica: Sequence[int],
                         devices: Sequence[int], cfg: Optional["CostModelConfig"] = None,
                         resident_weight_bytes: Optional[Sequence[float]] = None) -> dict:
        """task_cost_detail of one resolved task: agg (TaskCost), stage pieces
        [dp][pp] of (comp, tp, pp, hbm), bubble_replica."""
        sl = _arr(C.c_int32, stage_layers)
        nm = _arr(C.c_int64, nm_replica)
        dv = _arr(C.c_int32, devices)
        t = _ResolvedTask(task_slot, dp, pp, tp, sl, nm, dv)
        agg = (C.c_double * 7)()
        stage = (C.c_double * (4 * dp * pp))()
        bub = (C.c_double * dp)()
        res = _arr(C.c_double, resident_weight_bytes) if resident_weight_bytes is not None else None
        cc = (cfg or CostModelConfig())._c()
        err = C.create_string_buffer(1024)
        _raise(self.lib.hpg_task_cost(self._h, C.byref(t), C.byref(cc), res, agg, stage, bub, err,
                                      1024), err)
        keys = ("comp", "tp", "pp", "dp", "bubble", "hbm", "total")
        return {"agg": dict(zip(keys, list(agg))),
                "stage": [[tuple(stage[4 * (i * pp + j): 4 * (i * pp + j) + 4]) for j in range(pp)]
                          for i in range(dp)],
                "bubble_replica": list(bub)}

    def min_ring_bottleneck(self, devices: Sequence[int], volume_bytes: float) -> float:
        out = C.c_double()
        err = C.create_string_buffer(1024)
        _raise(self.lib.hpg_ring_bottleneck(self._h, _arr(C.c_int32, devices), len(devices),
                                            volume_bytes, C.byref(out), err, 1024), err)
        return out.value

    def min_pair_cost(self, src: Sequence[int], dst: Sequence[int], volume_bytes: float) -> float:
        out = C.c_double()
        err = C.create_string_buffer(1024)
        _raise(self.lib.hpg_pair_cost(self._h, _arr(C.c_int32, src), len(src),
                                      _arr(C.c_int32, dst), len(dst), volume_bytes, C.byref(out),
                                      err, 1024), err)
        return out.value

    def sweep_dist(self, seed: int, total: int, rank: int, world: int,
                   nccl_id: Optional[bytes] = None) -> dict:
        """hpg_sweep_dist: this rank's contiguous shard of [0, total), global argmin
        merged over the ranks with one NCCL all-gather."""
        st = _SweepStats()
        err = C.create_string_buffer(1024)
        idb = (C.c_uint8 * 128)(*(nccl_id or bytes(128)))
        rc = self.lib.hpg_sweep_dist(self._h, seed, total, rank, world, idb, C.byref(st), err,
                                     1024)
        _raise(rc, err)
        return {f: getattr(st, f) for f, _ in _SweepStats._fields_}

    def sweep_resident(self, seed: int, k0: int, count: int) -> dict:
        st = _SweepStats()
        err = C.create_string_buffer(1024)
        rc = self.lib.hpg_sweep_resident(self._h, seed, k0, count, C.byref(st), err, 1024)
        _raise(rc, err)
        return {f: getattr(st, f) for f, _ in _SweepStats._fields_}


class SearchResult:
    """SearchResult (search.hpp:105-111) read out of an hpg_search_result."""

    def __init__(self, eng: Engine, handle):
        lib = eng.lib
        info = _SearchInfo()
        lib.hpg_result_info(handle, C.byref(info))
        self.info = {f: getattr(info, f) for f, _ in _SearchInfo._fields_}
        self.consumed = info.consumed
        n = info.n_b_m
        b = (C.c_int64 * max(1, n))()
        lib.hpg_result_b_m(handle, b)
        self.b_m = [b[i] for i in range(n)]
        n = info.n_trace
        tc, tv = (C.c_int64 * max(1, n))(), (C.c_double * max(1, n))()
        lib.hpg_result_trace(handle, tc, tv)
        self.trace = [(tc[i], tv[i]) for i in range(n)]
        n = info.n_arms
        a1, a2, a3, a4 = ((C.c_int64 * max(1, n))(), (C.c_int64 * max(1, n))(),
                          (C.c_double * max(1, n))(), (C.c_int64 * max(1, n))())
        lib.hpg_result_arms(handle, a1, a2, a3, a4)
        self.arms = [(a1[i], a2[i], a3[i], a4[i]) for i in range(n)]
        n = info.n_halvings
        h1, h2, h3, h4, h5 = ((C.c_int32 * max(1, n))(), (C.c_int64 * max(1, n))(),
                              (C.c_int64 * max(1, n))(), (C.c_double * max(1, n))(),
                              (C.c_double * max(1, n))())
        lib.hpg_result_halvings(handle, h1, h2, h3, h4, h5)
        self.halvings = [(h1[i], h2[i], h3[i], h4[i], h5[i]) for i in range(n)]
        n = info.n_survivor_sets
        sz = (C.c_int32 * max(1, n))()
        lib.hpg_result_survivor_sizes(handle, sz)
        tot = sum(sz[i] for i in range(n))
        ix = (C.c_int64 * max(1, tot))()
        lib.hpg_result_survivors(handle, ix)
        self.survivors, k = [], 0
        for i in range(n):
            self.survivors.append([ix[k + j] for j in range(sz[i])])
            k += sz[i]
        self.plan = None
        self.breakdown = None
        if info.has_plan:
            pt = _PlanTable()
            T = len(eng.wf.tasks)
            gf = (C.c_int32 * T)()
            est, ps, pb = C.c_double(), C.c_uint64(), C.c_int64()
            lib.hpg_result_plan(handle, C.byref(pt), gf, C.byref(est), C.byref(ps), C.byref(pb))
            ids = eng.wf.task_ids
            ng = pt.n_groups[0]
            groups = [[] for _ in range(ng)]
            for s in gf:
                groups[pt.task_group[s]].append(ids[s])
            plan = dict(groups=groups, counts=[pt.gpu_counts[g] for g in range(ng)],
                        layouts={}, assignment={}, estimated_cost_s=est.value,
                        provenance=dict(seed=ps.value, budget=pb.value))
            for t, tid in enumerate(ids):
                dp_, pp_, tp_ = pt.dp[t], pt.pp[t], pt.tp[t]
                so, wo, do = pt.sl_off[t], pt.w_off[t], pt.dev_off[t]
                plan["layouts"][tid] = dict(dp=dp_, pp=pp_, tp=tp_,
                                            stage_layers=[pt.stage_layers[so + j]
                                                          for j in range(pp_)],
                                            weights=[pt.weights[wo + j] for j in range(dp_)])
                plan["assignment"][tid] = [pt.devices[do + j] for j in range(dp_ * pp_ * tp_)]
            self.plan = plan
            ptk = (C.c_double * (T * 7))()
            rs, sy, e2, mf = C.c_double(), C.c_double(), C.c_double(), C.c_uint8()
            lib.hpg_result_breakdown(handle, ptk, C.byref(rs), C.byref(sy), C.byref(e2),
                                     C.byref(mf))
            self.breakdown = dict(
                per_task={ids[t]: {COMPONENTS[c_]: ptk[t * 7 + c_] for c_ in range(7)}
                          for t in range(T)},
                reshard_s=rs.value, sync_s=sy.value, end_to_end_s=e2.value,
                memory_feasible=bool(mf.value))
        lib.hpg_result_free(handle)


def dist_exchange(rank: int, world: int, allgather, slices: Sequence[int],
                  used: Sequence[int], best: Sequence[float], mine) -> dict:
    """hpg_dist_exchange: the per-round record exchange of the sharded search
    over a Python all-gather `allgather(send: bytes) -> bytes` (world * len in
    rank order), e.g. torch.distributed over gloo. `mine` = [(run, local_idx,
    cost)] of this rank's runs; used/best entries of other ranks' runs are
    ignored. Returns owners, used, best and every run's improvements."""
    lib = load_library()
    n = len(slices)

    def cb(_user, send, recv, nbytes):
        try:
            out = allgather(C.string_at(send, nbytes) if nbytes else b"")
            if len(out) != nbytes * world:
                return 1
            if nbytes:
                C.memmove(recv, out, len(out))
            return 0
        except Exception:  # surfaced as a non-zero status
            return 1

    fn = ALLGATHER_FN(cb)
    sl = _arr(C.c_int64, slices)
    own = (C.c_int32 * max(1, n))()
    us = _arr(C.c_int64, used)
    bs = _arr(C.c_double, best)
    mi = (_Improvement * max(1, len(mine)))(*[_Improvement(*m) for m in mine])
    cap = 1 << 16
    al = (_Improvement * cap)()
    n_all = C.c_int64()
    err = C.create_string_buffer(1024)
    rc = lib.hpg_dist_exchange(rank, world, fn, None, n, sl, own, us, bs, mi, len(mine), al, cap,
                               C.byref(n_all), err, 1024)
    _raise(rc, err)
    return {"owner": list(own)[:n], "used": list(us)[:n], "best": list(bs)[:n],
            "impr": [(al[i].run, al[i].local_idx, al[i].cost) for i in range(n_all.value)]}

