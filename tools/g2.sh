cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_real_configs.py -q -s --durations=20 > $O/pytest_real.log 2>&1; echo "rc=$?" >> $O/pytest_real.log
