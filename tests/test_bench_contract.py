"""CPU checks of bench.py's workload definition (no GPU): the timed window
is centred on the BASELINE config's whole decode, so tokens/s is the full
decode's mean (step bytes are linear in n); the algorithmic bytes mirror
attend_algo_bytes in skv_capi.cu."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


@pytest.mark.parametrize("config", [2, 3])
@pytest.mark.parametrize("K", [1, 10, 50, 51, 200])
def test_timed_window_is_centred(config, K):
    cfg = bench.CONFIGS[config]
    s, dec = cfg["s"], cfg["decode"]
    W, n_first = bench.timed_window(cfg, 5, K)
    assert W >= 5 and n_first == s + W + 1
    mean = n_first + (K - 1) / 2.0
    assert abs(mean - (s + (dec + 1) / 2.0)) <= 0.5  # the window's mean n is the decode's
    assert s + 1 <= n_first and n_first + K - 1 <= s + dec


def test_timed_window_without_decode_length():
    cfg = bench.CONFIGS[4]  # steady state at KV length 4096
    assert bench.timed_window(cfg, 5, 50) == (5, cfg["s"] + 6)
    cfg2 = bench.CONFIGS[2]
    W, n_first = bench.timed_window(cfg2, 3, 600)  # longer than the decode: no centring
    assert (W, n_first) == (3, cfg2["s"] + 4)


def test_algo_bytes_config2():
    # n = 768: k = RNE(76.8) = 77, m = 154; f16 rows of 256 B, B=64, H=32
    cfg = bench.CONFIGS[2]
    H, B, row = 32, 64, 256
    want = B * (H * 128 * 2 * 2 + 2 * H * 128 * 2 + 2 * H * row + 2 * 153 * H * row)
    assert bench.attend_algo_bytes(cfg, 768) == want


@pytest.mark.parametrize("cfg_B,world,hs,want_B,want_seqs,want_scaling", [
    (64, 1, 0, 64, 64, "weak"),     # config 2 on one GPU
    (64, 8, 0, 64, 512, "weak"),    # batch-sharded: each GPU its own 64 sequences
    (1, 8, 0, 1, 1, "strong"),      # config 1: head shards over 8 GPUs, one sequence
    (1, 8, 8, 1, 1, "strong"),      # the same mesh named explicitly: same workload
    (16, 8, 2, 32, 128, "weak"),    # config 3: 4 groups x 32 sequences = b=128
    (16, 2, 2, 16, 16, "strong"),   # one group over 2 head shards: the 1-GPU batch
])
def test_mesh_workload(cfg_B, world, hs, want_B, want_seqs, want_scaling):
    """the implicit and explicit forms of the same mesh decode the
    same sequences, and `scaling` follows whether the global batch grew."""
    for rank in range(world):
        mw = bench.mesh_workload(cfg_B, world, rank, hs)
        assert (mw["B"], mw["seqs"], mw["scaling"]) == (want_B, want_seqs, want_scaling)
