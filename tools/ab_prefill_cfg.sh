# A/B of prefill library variants on the three MoE configs at batch 256: VARIANTS="a b" bash tools/ab_prefill_cfg.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O; rm -f $O/ab_cfg.txt
for r in 1 2; do for v in "" $VARIANTS; do for c in mixtral deepseek arctic; do
  MILO_B200_LIB_VARIANT=$v timeout 300 python tools/timeline.py --batch 256 --config $c > $O/tl.txt 2>&1
  echo "${v:-default} $c $(grep 'pf_gemm' $O/tl.txt | head -2 | sed 's/.*dur= *//; s/us.*//' | tr '\n' ' ') span $(grep 'layer span' $O/tl.txt)" >> $O/ab_cfg.txt
done; done; done
