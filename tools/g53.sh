cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -x -q > $O/pt_moe.txt 2>&1
tail -1 $O/pt_moe.txt
for v in "" nopf "" nopf; do for c in mixtral deepseek; do MILO_B200_LIB_VARIANT=$v timeout 300 python bench.py --config $c --no-cpu --no-parity --no-sweep --steps 30 > $O/b_${c}_$v.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/b_${c}_$v.json').read().strip().splitlines()[-1]); print('$c', '$v', d['value'], d['roofline']['frac'])" >> $O/pf_ab.txt; done; done
