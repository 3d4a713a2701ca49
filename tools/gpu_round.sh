#!/usr/bin/env bash
# One GPU session: parity tests, bench, timeline, launch list, ncu capture of the top kernel.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
mkdir -p $O
nvidia-smi -L > $O/gpu.txt 2>&1
nproc >> $O/gpu.txt; lscpu | grep "Model name" >> $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python tools/timeline.py --batch 1 > $O/timeline_m1.txt 2>&1
timeout 300 python tools/timeline.py --batch 256 > $O/timeline_m256.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_w3a16_kernel -s 6 -c 2 \
  -o $O/prof_gemv python tools/timeline.py --batch 1 --iters 2 > $O/ncu_full.log 2>&1
