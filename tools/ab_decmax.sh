cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; rm -f $O/decmax.txt
for b in 24 32 48 64; do for dm in 64 16; do echo "batch $b dec_max $dm $(MILO_DEC_MAX_M=$dm timeout 300 python tools/timeline.py --batch $b 2>&1 | grep 'layer span')" >> $O/decmax.txt; done; done
