cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; rm -f $O/ng2.txt
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_real_configs.py -x -q > $O/pt.txt 2>&1
for r in 1 2; do for v in 1 0; do for c in mixtral deepseek arctic; do
  echo "ng2=$v $c $(MILO_PF_NG2=$v timeout 300 python tools/timeline.py --batch 256 --config $c 2>&1 | grep 'pf_gemm_kernel<1\|layer span' | sed 's/start=.*dur=//' | tr '\n' ' ')" >> $O/ng2.txt
done; done; done
