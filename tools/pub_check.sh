cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/pub_pytest.log 2>&1; echo "rc=$?" >> $O/pub_pytest.log
for r in 1 2 3; do timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value',d['value'],[(s['batch'],s['us']) for s in d.get('sweep') or []])" >> $O/pub.txt; done
timeout 300 python tools/timeline.py --batch 256 2>/dev/null | head -4 >> $O/pub.txt
