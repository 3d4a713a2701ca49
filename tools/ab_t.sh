cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_moe.py tests/test_gpu_linear.py -m gpu -x -q > $O/ab_pytest.log 2>&1; echo "rc=$?" >> $O/ab_pytest.log
for r in 1 2; do for v in "" tv1; do
 echo "== variant '$v' run $r" >> $O/ab_t.txt
 MILO_B200_LIB_VARIANT=$v timeout 300 python tools/timeline.py --batch 256 2>/dev/null | grep -E "pf_img_t_kernel|layer span" | head -3 >> $O/ab_t.txt
 MILO_B200_LIB_VARIANT=$v timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value',d['value'],[(s['batch'],s['us']) for s in d.get('sweep') or []])" >> $O/ab_t.txt
done; done
