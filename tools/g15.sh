cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
HD_FLAGS=4 python tools/hd_timeline.py mixtral 1 > $O/hdt_nocopy.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hdec_kernel -s 3 -c 1 -o $O/prof_hd_mix1b -f python tools/hd_run.py mixtral 1 5 > $O/ncu_hd.log 2>&1
