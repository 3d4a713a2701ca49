cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
for f in 0 1; do MILO_B200_LIB_VARIANT=prof timeout 300 python tools/pf_stage_trace.py --batch 256 --flags $f > $O/pr256_$f.txt 2>&1; done
MILO_B200_LIB_VARIANT=prof timeout 300 python tools/pf_stage_trace.py --batch 2048 > $O/pr2048.txt 2>&1
