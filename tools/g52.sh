cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
for v in "" g4; do MILO_B200_LIB_VARIANT=$v timeout 300 python tools/timeline.py --batch 256 > $O/tl256_$v.txt 2>&1; MILO_B200_LIB_VARIANT=$v timeout 300 python tools/time_prefill.py 256 2048 > $O/tp_$v.txt 2>&1; done
