cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
python tools/pf_stage_trace.py --batch 256 > $O/st256.txt 2>&1
python tools/pf_stage_trace.py --batch 256 --flags 1 > $O/st256_f1.txt 2>&1
python tools/pf_stage_trace.py --batch 256 --flags 3 > $O/st256_f3.txt 2>&1
python tools/pf_stage_trace.py --batch 2048 --config mixtral > $O/st2048.txt 2>&1
python tools/timeline.py --batch 256 > $O/tl256.txt 2>&1
