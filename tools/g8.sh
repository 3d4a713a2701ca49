cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q -k "mixtral_like and (1 or 3 or 8 or 16)" > $O/pt_hd1.log 2>&1; echo "rc=$?" >> $O/pt_hd1.log
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_real_configs.py -q > $O/pt_hd2.log 2>&1; echo "rc=$?" >> $O/pt_hd2.log
for c in mixtral deepseek arctic; do
timeout 300 python bench.py --no-cpu --no-sweep --steps 20 --config $c > $O/b_hd_$c.json 2>$O/b_hd_$c.err
MILO_HDEC=0 timeout 300 python bench.py --no-cpu --no-sweep --no-parity --steps 20 --config $c > $O/b_old_$c.json 2>/dev/null
done
