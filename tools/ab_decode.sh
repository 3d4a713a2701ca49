# A/B of decode-kernel library variants at batch 1: VARIANTS="a b" bash tools/ab_decode.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O; rm -f $O/ab_decode.txt
for r in 1 2; do for v in "" $VARIANTS; do for c in mixtral deepseek; do MILO_B200_LIB_VARIANT=$v timeout 300 python bench.py --config $c --no-cpu --no-parity --no-sweep --steps 30 > $O/b.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$c', '${v:-default}', d['value'], d['roofline']['frac'])" >> $O/ab_decode.txt; done; done; done
