cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
HD_FLAGS=4 python tools/hd_timeline.py mixtral 1 > $O/hdt_f4.txt 2>&1
HD_FLAGS=12 python tools/hd_timeline.py mixtral 1 > $O/hdt_f12.txt 2>&1
