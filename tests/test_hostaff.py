"""Host NUMA placement helper of the e2e path (paper_2403_17312_b200/hostaff.py): cpulist parsing, and the
affinity bind is scoped to the allocation (restored after, a no-op when the GPU's node is unknown)."""
import os

from paper_2403_17312_b200 import hostaff


def test_cpulist_parsing():
    assert hostaff._cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert hostaff._cpulist("5") == [5]
    assert hostaff._cpulist("") == []


def test_near_gpu_binds_then_restores(monkeypatch):
    before = os.sched_getaffinity(0)
    one = sorted(before)[:1]
    monkeypatch.setattr(hostaff, "gpu_local_cpus", lambda device=0: one)
    with hostaff.near_gpu(0) as cpus:
        assert cpus == one
        assert os.sched_getaffinity(0) == set(one)
    assert os.sched_getaffinity(0) == before


def test_near_gpu_unknown_node_is_noop(monkeypatch):
    before = os.sched_getaffinity(0)
    monkeypatch.setattr(hostaff, "gpu_local_cpus", lambda device=0: None)
    with hostaff.near_gpu(0) as cpus:
        assert cpus is None
        assert os.sched_getaffinity(0) == before
