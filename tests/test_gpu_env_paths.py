"""GPU parity of the code paths selected by process-wide switches, each in a fresh
process (tests/env_parity_main.py):

* the default build at shapes the prefill kernel cannot take (f % 128 == 64) beyond the
  decode megakernel's batch: routed to token-chunked decode-megakernel calls;
* MILO_LEGACY=1, the round-1 multi-launch path (A/B reference, reachable only this way);
* MILO_HDEC=1, the h-local decode kernel (hdec.cuh, K4; opt-in).

Tolerances as tests/test_gpu_moe.py: layer output 1e-4 relative Frobenius (f32 in/out),
1e-3 for binary16 in/out; routing ids bit-exact; linear 1e-5.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(env_extra, cases):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    env.update(env_extra)
    res = subprocess.run([sys.executable, os.path.join(HERE, "env_parity_main.py"), *cases], env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert res.stdout.strip().endswith("ok")


def test_non_prefill_shapes_chunk_through_decode_kernel():
    _run({}, ["nonpf"])


def test_legacy_multi_launch_path():
    _run({"MILO_LEGACY": "1"}, ["mixtral", "nonpf", "linear"])


def test_h_local_decode_kernel():
    _run({"MILO_HDEC": "1"}, ["mixtral", "deepseek"])
