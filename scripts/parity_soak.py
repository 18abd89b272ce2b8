"""Parity soak: many seeded decode trajectories against the oracle (the
test suite's run_trajectory), across the BASELINE dtypes and head counts.
Prints the number of trajectories, steps and tolerated tie flips.

    python scripts/parity_soak.py [--seeds 12]
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import Oracle  # noqa: E402  (test infrastructure: the checker)
from test_gpu_parity import run_trajectory  # noqa: E402

from paper_2403_17312_b200 import api  # noqa: E402

CASES = [  # (dtype, B, H, s, steps, r)
    ("f32", 2, 32, 300, 12, 0.2),
    ("f16", 4, 32, 500, 12, 0.2),
    ("bf16", 2, 40, 600, 10, 0.2),
    ("u8", 2, 56, 700, 8, 0.2),
    ("f16", 3, 8, 200, 20, 0.05),
    ("f16", 2, 8, 120, 20, 0.5),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=12)
    args = ap.parse_args()
    port = Oracle("port")
    api.lib()
    total_traj = total_steps = total_flips = 0
    for dt, B, H, s, steps, r in CASES:
        flips = 0
        for seed in range(args.seeds):
            flips += run_trajectory(api, port, dt, B, H, s, steps, r, seed=10_000 + seed)
        total_traj += args.seeds * B
        total_steps += args.seeds * B * steps
        total_flips += flips
        print(f"{dt:4s} B={B} H={H} s={s} steps={steps} r={r}: {args.seeds} seeds, tie flips {flips}", flush=True)
    print(f"ALL: {total_traj} sequence trajectories, {total_steps} decode steps, {total_flips} tolerated tie flips")


if __name__ == "__main__":
    main()
