cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw,clocks_throttle_reasons.active --format=csv > $O/sweep_dbg.txt
for r in 1 2 3; do
 echo "== run $r" >> $O/sweep_dbg.txt
 MILO_BENCH_DUMP_STEPS=1 timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 2>>$O/sweep_dbg.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value',d['value'],d['clocks'],[(s['batch'],s['us']) for s in d.get('sweep') or []])" >> $O/sweep_dbg.txt
done
timeout 300 python tools/timeline.py --batch 16 --iters 3 > $O/timeline_m16.txt 2>&1
