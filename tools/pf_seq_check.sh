cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/seq_pytest.log 2>&1; echo "rc=$?" >> $O/seq_pytest.log
timeout 300 python tools/timeline.py --batch 256 > $O/seq_timeline.txt 2>&1
MILO_HOST_PROF=1 timeout 300 python tools/timeline.py --batch 256 --iters 3 2>&1 | grep "moe_prefill host" | tail -8 > $O/seq_hostprof.txt
for r in 1 2; do timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value',d['value'],'e2e',d['e2e']['value'],[(s['batch'],s['us']) for s in d.get('sweep') or []])" >> $O/seq_bench.txt; done
