cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pf_gemm_kernel -c 1 -o $O/pf256b python tools/moe_once.py --batch 256 > $O/ncu_pf256.log 2>&1
MILO_B200_LIB_VARIANT=as4 timeout 300 python tools/timeline.py --batch 256 > $O/tl256_as4.txt 2>&1
