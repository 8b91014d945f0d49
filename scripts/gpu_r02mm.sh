#!/usr/bin/env bash
# round 2 (final build): the GPU parity suite on the bounds-checked build, plus one memcheck attempt
cd "$(dirname "$0")/.."
O=gpurun_out
HPG_LIBRARY=$PWD/paper_2512_12476_b200/libhpg_checked.so timeout 2400 python -m pytest tests/test_gpu_parity.py -q -rs > $O/r02mm_checked_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02mm_checked_pytest.txt
HPG_LIBRARY=$PWD/paper_2512_12476_b200/libhpg_checked.so HPG_DEVICE_GA=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "search_configs or search_fuzz" > $O/r02mm_checked_hostga.txt 2>&1; echo "rc=$?" >> $O/r02mm_checked_hostga.txt
HPG_LIBRARY=$PWD/paper_2512_12476_b200/libhpg_checked.so timeout 300 python scripts/sweep_probe.py 2000000 > $O/r02mm_checked_sweep.jsonl 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/search_probe.py c1 1000 0 1 > $O/r02mm_memcheck.txt 2>&1; echo "rc=$?" >> $O/r02mm_memcheck.txt
