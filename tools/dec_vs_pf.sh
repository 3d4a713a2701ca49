cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O; : > $O/dvp.txt
for c in mixtral deepseek; do for b in 1 48 64; do for env in 64; do
 v=$(MILO_DEC_MAX_M=$env timeout 300 python bench.py --config $c --batch $b --no-cpu --no-sweep --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'])")
 echo "$c batch $b dec_max_m $env: $v" >> $O/dvp.txt
done; done; done
