#!/usr/bin/env bash
# round 2: per-plan phase cycles of c4 evaluations (host-GA path: eval_kernel waves)
cd "$(dirname "$0")/.."
O=gpurun_out
CFGS=c4 HPG_DEVICE_GA=0 bash scripts/gpu_planprof.sh > $O/r02v_planprof.log 2>&1
python scripts/planprof_summary.py gpurun_out/planprof_c4.txt.gz 20 > $O/r02v_planprof_summary.txt 2>&1
python scripts/planprof_phases.py gpurun_out/planprof_c4.txt.gz > $O/r02v_planprof_phases.txt 2>&1
