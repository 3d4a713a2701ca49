# A/B of library variants on the bench (default workload + sweep): tools/ab.sh v1 v2 ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
for v in "$@"; do
  if [ "$v" = base ]; then unset MILO_B200_LIB_VARIANT; else export MILO_B200_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --no-cpu --steps 30 > $O/ab_$v.json 2> $O/ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{v}.json"))
    print(f"{v:10s} value {d['value']:8.2f} us  e2e {d['e2e']['value']:8.2f}  parity {d['parity']['rel_err']:.2e}  sweep " +
          " ".join(f"{s['batch']}:{s['us']:.1f}" for s in d['sweep']))
except Exception as e:
    print(v, "failed", e, open(f"gpurun_out/ab_{v}.err").read()[-800:])
PY
done
