#!/usr/bin/env bash
# Regenerates every golden fixture in tests/golden/ from the UNMODIFIED
# reference planner (compiled from /root/reference by oracle/Makefile into
# oracle/_ref/ref_dump). Runs in the build container only (needs
# /root/reference); the GPU box uses the committed JSON.
set -euo pipefail
cd "$(dirname "$0")/../.."
make -C oracle ref
R=oracle/_ref/ref_dump
G=tests/golden
KNOBS=/root/reference/proj/samples/knobs.json
for c in c1 c2; do
  $R evalplans fixtures/$c.workflow.json fixtures/$c.topology.json 42 60 $G/evalplans_$c.json
done
for c in c3 c4; do
  $R evalplans fixtures/$c.workflow.json fixtures/$c.topology.json 42 24 $G/evalplans_$c.json
done
# 256 GPUs, 4 types x 8 regions (the engine's device-index limit); topology
# from the fleet generator: hetplan_b200 scenario --id fleet --gpus
# 64xA100,64xL40S,64xL4,64xH100 --regions virginia,ohio,paris,frankfurt,tokyo,
# sydney,saopaulo,mumbai --seed 3 (byte-identical to the committed fixture)
$R evalplans fixtures/n256.workflow.json fixtures/n256.topology.json 7 16 $G/evalplans_n256.json
$R fuzz 20251018 250 $G/fuzz_eval.json
$R search fixtures/c1.workflow.json fixtures/c1.topology.json 1000 42 $G/search_c1_b1000.json $KNOBS
$R search fixtures/c2.workflow.json fixtures/c2.topology.json 1000 42 $G/search_c2_b1000.json $KNOBS
# every search config at both parity budgets (B in {10^3, 10^4})
for c in c3 c4; do
  $R search fixtures/$c.workflow.json fixtures/$c.topology.json 1000 42 $G/search_${c}_b1000.json $KNOBS
done
for c in c1 c2 c3 c4; do
  $R search fixtures/$c.workflow.json fixtures/$c.topology.json 10000 42 $G/search_${c}_b10000.json $KNOBS
done
$R search fixtures/n256.workflow.json fixtures/n256.topology.json 1000 42 $G/search_n256_b1000.json $KNOBS
$R searchfuzz 777 60 $G/searchfuzz.json
for c in c1 c2 c3 c4; do
  $R ga fixtures/$c.workflow.json fixtures/$c.topology.json $G/ga_$c.json $KNOBS
done
$R sweep fixtures/c4.workflow.json fixtures/c4.topology.json 42 0 2000 $G/sweep_c4.json
$R exhaustive 4242 40 $G/exhaustive.json
python3 - <<'PY'
import json, subprocess
out = {}
for seed in ("42", "0", "18446744073709551615", "20251018"):
    r = subprocess.run(["oracle/_ref/ref_dump", "rngpin", seed], capture_output=True, text=True,
                       check=True)
    out[seed] = r.stdout.strip().splitlines()
json.dump(out, open("tests/golden/rng_pin.json", "w"), indent=1)
PY
$R cli $G/cli/cases.json
