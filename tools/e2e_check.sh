cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_moe.py -m gpu -x -q > $O/e2e_pytest.log 2>&1; echo "rc=$?" >> $O/e2e_pytest.log
for r in 1 2; do timeout 300 python bench.py --no-cpu --no-sweep --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value',d['value'],'e2e',d['e2e'])" >> $O/e2e.txt; done
