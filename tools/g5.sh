cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_real_configs.py -x -q > $O/pt_plan.log 2>&1; echo "rc=$?" >> $O/pt_plan.log
timeout 600 python bench.py --no-cpu --steps 20 > $O/bench_plan.json 2>/dev/null
python -c "import json,sys; d=json.load(open('$O/bench_plan.json')); print([(s['batch'], s['us']) for s in d['sweep']])"
timeout 300 python tools/timeline.py --batch 256 > $O/timeline_m256.txt 2>&1
