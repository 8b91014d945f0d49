#!/usr/bin/env bash
# round 2: sweep ordering key v2 (training tasks first, half-octave, bridge class)
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep" > $O/r02j_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02j_pytest.txt
for i in 1 2; do timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02j_sweep.jsonl 2>> $O/r02j_sweep.err; done
HPG_SWEEP_SYNC=2 timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02j_sweep.jsonl 2>> $O/r02j_sweep.err
