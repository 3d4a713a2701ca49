# A/B of prefill library variants: VARIANTS="a b" bash tools/ab_prefill.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O; rm -f $O/ab_prefill.txt
for r in 1 2 3; do for v in "" $VARIANTS; do
  MILO_B200_LIB_VARIANT=$v timeout 300 python tools/timeline.py --batch 256 > $O/tl.txt 2>&1
  echo "${v:-default} $(grep 'pf_gemm' $O/tl.txt | head -2 | sed 's/.*dur= *//; s/us.*//' | tr '\n' ' ') span $(grep 'layer span' $O/tl.txt)" >> $O/ab_prefill.txt
done; done
