cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
python tools/time_prefill.py 2048 > $O/tp.txt 2>&1
python tools/time_prefill.py 256 >> $O/tp.txt 2>&1
for f in 3 0; do PF_FLAGS=$f python tools/dbg_pf_timeline.py 2048 > $O/pft_$f.txt 2>&1; done
timeout 600 python bench.py --no-cpu --steps 20 > $O/bench_pf.json 2>/dev/null
