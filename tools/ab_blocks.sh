cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/abb_pytest.log 2>&1; echo "rc=$?" >> $O/abb_pytest.log
for r in 1 2; do for v in "" tvp0; do for c in mixtral deepseek; do
 echo "== variant '$v' $c run $r" >> $O/abb.txt
 MILO_B200_LIB_VARIANT=$v timeout 300 python bench.py --config $c --no-cpu --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value',d['value'],[(s['batch'],s['us']) for s in d.get('sweep') or []])" >> $O/abb.txt
done; done; done
