"""Sharded-search scaling probe (not the bench): under torchrun with N ranks
(or plain python for N = 1), run `warm` + `runs` searches of (config, budget)
and print rank 0's JSON line: device-timed ms per search (max over ranks),
plans/s, and the chosen cost (identical on every rank).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      scripts/dist_scale.py c4 100000
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from paper_2512_12476_b200 import Engine, SearchKnobs, distutil, load_topology, load_workflow  # noqa

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 1
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 3
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
K = dict(budget=budget, seed=42, population=16, locality_bias=0.8, quantize_gpu_counts=1,
         level1_filter="off", gg_arm_cap=64, swap_pair_sample=8, balance_data=True,
         balance_layers=True, balance_seqlen=True, recompute=True)
eng = Engine(load_workflow(f"{ROOT}/fixtures/{cfg}.workflow.json"),
             load_topology(f"{ROOT}/fixtures/{cfg}.topology.json"), device=local)
k = SearchKnobs.from_json(K)
nid = None
if world > 1:
    nid = distutil.broadcast_bytes(eng.nccl_unique_id() if rank == 0 else None, 0)


def search():
    return eng.nested_sha_search(k) if world == 1 else eng.nested_sha_search_dist(k, rank, world, nid)


for _ in range(warm):
    search()
ms, res = [], None
for _ in range(runs):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = search()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    ms.append(t if world == 1 else 1000.0 * distutil.max_over_ranks(t / 1000.0))
if rank == 0:
    print(json.dumps({"config": cfg, "budget": budget, "world": world, "ms": ms,
                      "plans_per_s": res.consumed / (min(ms) / 1000.0), "consumed": res.consumed,
                      "best": res.breakdown["end_to_end_s"] if res.breakdown else None}), flush=True)
eng.close()
if world > 1:
    dist.destroy_process_group()
