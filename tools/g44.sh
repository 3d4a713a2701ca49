cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_moe.py -x -q > $O/pt_lin_moe.txt 2>&1
tail -2 $O/pt_lin_moe.txt
for v in "" iss1 as4; do MILO_B200_LIB_VARIANT=$v timeout 300 python tools/timeline.py --batch 256 > $O/tl256_$v.txt 2>&1; MILO_B200_LIB_VARIANT=$v timeout 300 python tools/time_prefill.py 256 2048 > $O/tp_$v.txt 2>&1; done
