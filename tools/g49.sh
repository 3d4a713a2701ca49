cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
for c in deepseek arctic; do timeout 300 python tools/timeline.py --batch 256 --config $c > $O/tl256_$c.txt 2>&1; done
timeout 300 python tools/timeline.py --batch 64 --config arctic > $O/tl64_arctic.txt 2>&1
