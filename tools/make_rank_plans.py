"""Freezes the benchmark layers' compensator ranks as rank plans made by the reference
itself (oracle/_ref, ref_plan_synth in oracle/ref/ref_capi.cpp): per-matrix kurtosis of
the reference's synthetic StudentTMix expert weights (synth.cpp, stats.cpp) and
plan_ranks with the paper's policies (rank_policy.cpp:94-164):

  mixtral  : Kurtosis-16 over 8 experts x {w1, w2, w3}
  deepseek : Dense-512+Kurtosis-16 (64 routed experts; the 2 shared experts are dense)
  arctic   : Kurtosis-16 over 128 experts

Writes paper_2504_02658_b200/plans/<config>.plan.json in the reference's plan format
(save_plan, pipeline.cpp: {"policy", "ranks", "avg_sparse_rank"}), read by
artifacts.load_plan and used by synth.build_host_layer.  Needs /root/reference built into
oracle/_ref (oracle/build_ref.sh); the plans are committed, so the GPU box does not.

    python tools/make_rank_plans.py
"""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_02658_b200.synth import CONFIGS  # noqa: E402

PLANS = {
    # name: (policy, shared experts, synthesized stats shape or None for the model's)
    "mixtral": ("Kurtosis-16", 0, None),
    "deepseek": ("Dense-512+Kurtosis-16", 2, None),
    "arctic": ("Kurtosis-16", 0, (1024, 1024)),
}


def main():
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libmilo_ref.so"))
    f = lib.ref_plan_synth
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                  ctypes.c_uint64, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p]
    out_dir = os.path.join(ROOT, "paper_2504_02658_b200", "plans")
    os.makedirs(out_dir, exist_ok=True)
    for name, (policy, shared, stats_shape) in PLANS.items():
        spec = CONFIGS[name]
        E = spec.experts
        ranks = np.zeros((E + shared) * 3, np.int32)
        kurt = np.zeros(E * 3, np.float64)
        sr, sc = stats_shape if stats_shape else (0, 0)
        t0 = time.time()
        st = f(E, shared, spec.d, spec.f, sr, sc, 0, policy.encode(), ranks.ctypes.data, kurt.ctypes.data)
        if st != 0:
            raise SystemExit(f"{name}: ref_plan_synth failed ({st})")
        names = []
        for x in range(E + shared):
            pre = f"layer0.expert{x}." if x < E else f"layer0.shared_expert{x - E}."
            names += [pre + w for w in ("w1", "w3", "w2")]
        plan = {"policy": policy, "ranks": {n: int(r) for n, r in zip(names, ranks)},
                "avg_sparse_rank": float(ranks[:E * 3].mean()),
                "generated_by": "tools/make_rank_plans.py (reference plan_ranks over the reference's "
                                "synthetic StudentTMix expert weights, seed 0"
                                + (f", stats at {sr}x{sc}" if stats_shape else "") + ")",
                "kurtosis": {n: float(k) for n, k in zip(names[:E * 3], kurt)}}
        with open(os.path.join(out_dir, f"{name}.plan.json"), "w") as fh:
            json.dump(plan, fh, indent=1, sort_keys=True)
        print(f"{name}: {policy} avg {plan['avg_sparse_rank']:.2f}, ranks min {ranks[:E*3].min()} "
              f"max {ranks[:E*3].max()} ({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
