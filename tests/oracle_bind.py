"""ctypes binding of the C restatement oracle (oracle/hp_oracle.c).

TEST INFRASTRUCTURE ONLY: used by tests/ and smoke() as the checker. Builds
oracle/_ref/libhp_oracle.so on first use (plain gcc, no reference needed).
"""
import ctypes as C
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_ref", "libhp_oracle.so")
MAXT = 6

_lib = None


class Task(C.Structure):
    _fields_ = [("id", C.c_int), ("kind", C.c_int), ("prec", C.c_int), ("emb", C.c_int),
                ("h1", C.c_longlong), ("h2", C.c_longlong), ("nl", C.c_longlong),
                ("vocab", C.c_longlong)]


class Problem(C.Structure):
    _fields_ = [("n_dev", C.c_int), ("comp", C.POINTER(C.c_double)),
                ("mem", C.POINTER(C.c_double)), ("hbm", C.POINTER(C.c_double)),
                ("lat", C.POINTER(C.c_double)), ("bw", C.POINTER(C.c_double)),
                ("n_tasks", C.c_int), ("tasks", Task * MAXT), ("mode", C.c_int),
                ("eta", C.c_double), ("global_batch", C.c_longlong), ("rpp", C.c_longlong),
                ("seq_in", C.c_longlong), ("seq_out", C.c_longlong), ("mbs", C.c_longlong)]


class Cfg(C.Structure):
    _fields_ = [("recompute", C.c_int), ("reshard_override", C.c_double),
                ("sync_override", C.c_double), ("dbs_override", C.c_double),
                ("train_bpp", C.c_double), ("infer_bpp", C.c_double), ("kv_bpe", C.c_double),
                ("dbs_cap", C.c_int), ("act_factor", C.c_double)]


class Plan(C.Structure):
    _fields_ = [("dp", C.c_int * MAXT), ("pp", C.c_int * MAXT), ("tp", C.c_int * MAXT),
                ("sl", C.POINTER(C.c_int) * MAXT), ("w", C.POINTER(C.c_double) * MAXT),
                ("dev", C.POINTER(C.c_int) * MAXT)]


class Breakdown(C.Structure):
    _fields_ = [("per_task", (C.c_double * 7) * MAXT), ("reshard", C.c_double),
                ("sync", C.c_double), ("e2e", C.c_double), ("feasible", C.c_int)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "restatement"],
                           check=True, capture_output=True)
        L = C.CDLL(LIB)
        P = C.POINTER
        L.hpo_ring.restype = C.c_double
        L.hpo_ring.argtypes = [P(Problem), P(C.c_int), C.c_int, C.c_double]
        L.hpo_check_memory.restype = C.c_int
        L.hpo_check_memory.argtypes = [P(Problem), P(Cfg), P(Plan), P(C.c_double)]
        L.hpo_end_to_end.argtypes = [P(Problem), P(Cfg), P(Plan), P(Breakdown)]
        L.hpo_balance_data.argtypes = [P(Problem), P(Cfg), P(Plan)]
        L.hpo_balance_layers.argtypes = [P(Problem), P(Cfg), P(Plan)]
        L.hpo_evaluate.argtypes = [P(Problem), P(Cfg), P(Plan), P(Breakdown)]
        _lib = L
    return _lib


def _f(v):
    return float.fromhex(v) if isinstance(v, str) else float(v)


def link_matrix(topo):
    """DeviceTopology::make's link rules (topology.cpp:85-111), restated."""
    devs = topo["devices"]
    n = len(devs)
    d = topo.get("defaults", {})
    dl = _f(d.get("intra_region_latency_ms", 0.1)) * 1e-3
    dbw = _f(d.get("intra_region_bandwidth_gbps", 100.0)) * 1.25e8
    rl = {}
    for l in topo.get("region_links", []):
        key = tuple(sorted((l["src"], l["dst"])))
        rl[key] = (_f(l["latency_ms"]) * 1e-3, _f(l["bandwidth_gbps"]) * 1.25e8)
    lat, bw = [0.0] * (n * n), [0.0] * (n * n)
    for a in range(n):
        for b in range(n):
            A, B = devs[a], devs[b]
            if a == b:
                x, y = 0.0, float("inf")
            elif A["node"] == B["node"] and A["region"] == B["region"]:
                x, y = 5e-6, min(_f(A["intra_node_gbps"]) * 1e9, _f(B["intra_node_gbps"]) * 1e9)
            elif A["region"] == B["region"]:
                x, y = dl, dbw
            else:
                x, y = rl[tuple(sorted((A["region"], B["region"])))]
            lat[a * n + b], bw[a * n + b] = x, y
    return lat, bw


class Oracle:
    def __init__(self, wf, topo):
        self.L = lib()
        devs = topo["devices"]
        n = len(devs)
        lat, bw = link_matrix(topo)
        self._arr = [(C.c_double * n)(*[_f(d["comp_tflops"]) * 1e12 for d in devs]),
                     (C.c_double * n)(*[_f(d["mem_gb"]) * 1e9 for d in devs]),
                     (C.c_double * n)(*[_f(d["hbm_gbps"]) * 1e9 for d in devs]),
                     (C.c_double * (n * n))(*lat), (C.c_double * (n * n))(*bw)]
        p = Problem()
        p.n_dev = n
        p.comp, p.mem, p.hbm, p.lat, p.bw = self._arr
        self.ids = [t["id"] for t in wf["tasks"]]
        p.n_tasks = len(wf["tasks"])
        for i, t in enumerate(wf["tasks"]):
            p.tasks[i] = Task(t["id"], t["kind"], t["precision_bytes"], int(t["include_embedding"]),
                              t["hidden_size"], t["intermediate_size"], t["num_layers"],
                              t["vocab_size"])
        p.mode = 0 if wf["mode"] == "sync" else 1
        p.eta = _f(wf["eta"])
        b = wf["batch"]
        p.global_batch, p.rpp = b["global_batch"], b["responses_per_prompt"]
        p.seq_in, p.seq_out, p.mbs = b["seq_in"], b["seq_out"], b["micro_batch_size"]
        self.p = p

    @staticmethod
    def cfg(obj):
        m = obj.get("memory", {})
        return Cfg(int(obj.get("recompute", True)), _f(obj.get("reshard_override", -1.0)),
                   _f(obj.get("sync_override", -1.0)), _f(obj.get("dbs_override", -1.0)),
                   _f(m.get("train_bytes_per_param", 18.0)),
                   _f(m.get("infer_bytes_per_param", 2.0)), _f(m.get("kv_bytes_per_elem", 2.0)),
                   int(m.get("dbs_cap", 1)), _f(m.get("act_factor", 4.0)))

    def plan(self, gp):
        """hpo_plan from a golden plan dict; keeps the arrays alive on the object"""
        pl = Plan()
        keep = []
        for i, tid in enumerate(self.ids):
            l = gp["layouts"][str(tid)] if str(tid) in gp["layouts"] else gp["layouts"][tid]
            a = gp["assignment"][str(tid)] if str(tid) in gp["assignment"] else gp["assignment"][tid]
            pl.dp[i], pl.pp[i], pl.tp[i] = l["dp"], l["pp"], l["tp"]
            sl = (C.c_int * len(l["stage_layers"]))(*l["stage_layers"])
            w = (C.c_double * len(l["weights"]))(*[_f(x) for x in l["weights"]])
            dv = (C.c_int * len(a))(*a)
            keep += [sl, w, dv]
            pl.sl[i] = C.cast(sl, C.POINTER(C.c_int))
            pl.w[i] = C.cast(w, C.POINTER(C.c_double))
            pl.dev[i] = C.cast(dv, C.POINTER(C.c_int))
        pl._keep = keep
        return pl

    def layouts_of(self, pl):
        out = {}
        for i, tid in enumerate(self.ids):
            out[tid] = dict(stage_layers=[pl.sl[i][j] for j in range(pl.pp[i])],
                            weights=[pl.w[i][j] for j in range(pl.dp[i])])
        return out

    def e2e(self, pl, cfg):
        bd = Breakdown()
        self.L.hpo_end_to_end(C.byref(self.p), C.byref(cfg), C.byref(pl), C.byref(bd))
        return bd

    def check_memory(self, pl, cfg):
        req = (C.c_double * self.p.n_dev)()
        ok = self.L.hpo_check_memory(C.byref(self.p), C.byref(cfg), C.byref(pl), req)
        return bool(ok), list(req)

    def balance_data(self, pl, cfg):
        self.L.hpo_balance_data(C.byref(self.p), C.byref(cfg), C.byref(pl))

    def balance_layers(self, pl, cfg):
        self.L.hpo_balance_layers(C.byref(self.p), C.byref(cfg), C.byref(pl))

    def evaluate(self, pl, cfg):
        bd = Breakdown()
        self.L.hpo_evaluate(C.byref(self.p), C.byref(cfg), C.byref(pl), C.byref(bd))
        return bd
