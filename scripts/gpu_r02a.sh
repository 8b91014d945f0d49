#!/usr/bin/env bash
# round 2: GPU suite + first c4 bench line
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
nproc > gpurun_out/r02a_nproc.txt; lscpu >> gpurun_out/r02a_nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r02a_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a_pytest.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench.jsonl 2> gpurun_out/r02a_bench.err
echo "bench rc=$?" >> gpurun_out/r02a_bench.err
