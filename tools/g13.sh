cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
for f in 0 1 2; do HD_FLAGS=$f python tools/hd_timeline.py mixtral 1 > $O/hdt_mix1_f$f.txt 2>&1; done
