"""Multi-GPU search parity: run under torchrun with N ranks; every rank runs
the sharded nested SHA search and compares it with the reference golden
(identical trace, arm records, halvings, survivor sets, chosen plan).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      scripts/dist_check.py search_c2_b1000.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from golden_util import load  # noqa: E402
from test_gpu_parity import check_search  # noqa: E402
from paper_2512_12476_b200 import Engine, SearchKnobs, parse_topology, parse_workflow  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    names = sys.argv[1:] or ["search_c1_b1000.json", "search_c2_b1000.json",
                             "search_c2_b10000.json", "search_c4_b10000.json"]
    ok = True
    for name in names:
        g = load(name)
        eng = Engine(parse_workflow(g["workflow"]), parse_topology(g["topology"]), device=local)
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.tensor(list(eng.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        t0 = time.perf_counter()
        res = eng.nested_sha_search_dist(SearchKnobs.from_json(g["knobs"]), rank, world,
                                         bytes(idt.cpu().tolist()))
        dt = time.perf_counter() - t0
        bad = check_search(res, g, f"{name} rank {rank}")
        ok = ok and not bad
        print(json.dumps({"rank": rank, "world": world, "case": name, "ok": not bad,
                          "bad": bad[:3], "wall_s": dt, "consumed": res.consumed}), flush=True)
        eng.close()
    # sharded config-5 sweep (hpg_sweep_dist): global argmin / count / checksum
    # equal to one GPU sweeping the whole range
    from paper_2512_12476_b200 import load_topology, load_workflow
    fx = os.path.join(ROOT, "fixtures")
    eng = Engine(load_workflow(f"{fx}/c4.workflow.json"), load_topology(f"{fx}/c4.topology.json"),
                 device=local)
    idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        idt.copy_(torch.tensor(list(eng.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    total = 400000
    st = eng.sweep_dist(42, total, rank, world, bytes(idt.cpu().tolist()))
    one = eng.sweep_resident(42, 0, total)
    keys = ("best_cost", "best_k", "n_feasible", "xor_bits")
    sweep_ok = all(st[k] == one[k] for k in keys)
    ok = ok and sweep_ok
    print(json.dumps({"rank": rank, "world": world, "case": "sweep_dist", "ok": sweep_ok,
                      "dist": {k: st[k] for k in keys}, "single": {k: one[k] for k in keys}}),
          flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
