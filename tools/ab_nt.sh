# decode megakernel: 8-row (NT = 1) vs 16-row (NT = 2) variant by batch (MILO_DEC_NT1_MAX)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; rm -f $O/ab_nt.txt
for c in mixtral deepseek; do for b in 12 16 24 32; do for t in 8 64; do
  echo "$c batch $b nt1_max $t $(MILO_DEC_NT1_MAX=$t timeout 300 python tools/timeline.py --config $c --batch $b 2>&1 | grep 'layer span')" >> $O/ab_nt.txt
done; done; done
