#!/usr/bin/env bash
# Round-2 checkpoint: full GPU suite, smoke, bench (3 configs), timelines, launch list,
# ncu full captures of the MoE prefill kernels at batch 256.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${CHECKPOINT:-r02c}; mkdir -p $O
nvidia-smi -L > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_mixtral.json 2> $O/bench_mixtral.err
timeout 900 python bench.py --config deepseek --no-cpu > $O/bench_deepseek.json 2> $O/bench_deepseek.err
timeout 900 python bench.py --config arctic --no-cpu > $O/bench_arctic.json 2> $O/bench_arctic.err
timeout 300 python tools/timeline.py --batch 256 > $O/timeline_m256.txt 2>&1
timeout 300 python tools/time_prefill.py 256 512 2048 > $O/time_prefill.txt 2>&1
MILO_B200_LIB_VARIANT=prof timeout 300 python tools/pf_stage_trace.py --batch 256 > $O/stage_trace_m256.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pf_gemm_kernel -c 2 -o $O/ncu_pf_m256 python tools/moe_once.py --batch 256 > $O/ncu_pf.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_m256.csv python tools/moe_once.py --batch 256 --iters 2 > $O/ncu_launch.log 2>&1
