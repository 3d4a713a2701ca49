cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pf_t_kernel -c 1 -o $O/pft_ds python tools/moe_once.py --batch 256 --config deepseek > $O/ncu_pft.log 2>&1
