cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_real_configs.py tests/test_gpu_moe.py -q > $O/pt_plan2.log 2>&1; echo "rc=$?" >> $O/pt_plan2.log
for c in mixtral deepseek arctic; do
timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
