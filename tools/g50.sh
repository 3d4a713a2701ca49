cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_real_configs.py -x -q > $O/pt_moe.txt 2>&1
tail -2 $O/pt_moe.txt
for c in mixtral deepseek arctic; do timeout 300 python tools/timeline.py --batch 256 --config $c > $O/tl256_$c.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_linear.py -x -q > $O/pt_lin.txt 2>&1
tail -1 $O/pt_lin.txt
