cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pf_gemm_kernel -c 2 -o $O/pf256 python tools/moe_once.py --batch 256 > $O/ncu_pf256.log 2>&1
tail -3 $O/ncu_pf256.log
