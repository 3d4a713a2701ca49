cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
HD_FLAGS=20 python tools/hd_timeline.py mixtral 1 > $O/hdt_f20.txt 2>&1
python tools/hd_timeline.py mixtral 1 > $O/hdt_p.txt 2>&1
HD_FLAGS=4 python tools/hd_timeline.py mixtral 1 > $O/hdt_f4.txt 2>&1
