cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_real_configs.py tests/test_gpu_ep.py -x -q > $O/pt_plan.log 2>&1; echo "rc=$?" >> $O/pt_plan.log
for v in dev host dev host; do
  if [ $v = host ]; then export MILO_PF_HOSTPLAN=1; else unset MILO_PF_HOSTPLAN; fi
  timeout 600 python bench.py --no-cpu --steps 20 > $O/ab_plan_$v.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('$O/ab_plan_$v.json')); print('$v', [(s['batch'], s['us']) for s in d['sweep']], d['c1_linear']['sweep'][-1]['us'])"
done
unset MILO_PF_HOSTPLAN
timeout 300 python tools/timeline.py --batch 256 > $O/timeline_m256.txt 2>&1
