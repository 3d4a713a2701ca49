#!/usr/bin/env bash
# One GPU session: parity tests, smoke, bench, timelines, launch list, ncu captures of the
# decode megakernel (m = 1) and the tcgen05 prefill kernel (m = 256).
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
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 6 -c 1 \
  -o $O/prof_decode python tools/timeline.py --batch 1 --iters 3 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pf_gemm_kernel -s 3 -c 1 \
  -o $O/prof_prefill python tools/time_prefill.py 2048 >> $O/ncu_full.log 2>&1
