cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
for f in 0 4 8 12 13 2; do MILO_B200_LIB_VARIANT=prof timeout 300 python tools/pf_stage_trace.py --batch 256 --flags $f > $O/fl_$f.txt 2>&1; done
