cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
MILO_HDEC=1 python tools/hd_timeline.py mixtral 1 > $O/hdt_w.txt 2>&1
MILO_HDEC=1 HD_FLAGS=64 python tools/hd_timeline.py mixtral 1 > $O/hdt_w64.txt 2>&1
MILO_HDEC=1 timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_real_configs.py -x -q > $O/pt_hd2.log 2>&1; echo "rc=$?" >> $O/pt_hd2.log
for c in mixtral deepseek arctic; do
MILO_HDEC=1 timeout 300 python bench.py --no-cpu --no-sweep --steps 20 --config $c > $O/b_hd_$c.json 2>$O/b_hd_$c.err
done
