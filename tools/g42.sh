cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_moe.py -x -q > $O/pt_lin_moe.txt 2>&1
tail -2 $O/pt_lin_moe.txt
MILO_B200_LIB_VARIANT=prof timeout 300 python tools/pf_stage_trace.py --batch 256 > $O/pr256_0.txt 2>&1
timeout 300 python tools/timeline.py --batch 256 > $O/tl256.txt 2>&1
MILO_B200_LIB_VARIANT=as4 timeout 300 python tools/timeline.py --batch 256 > $O/tl256_as4.txt 2>&1
timeout 300 python tools/time_prefill.py 256 2048 > $O/tp.txt 2>&1
