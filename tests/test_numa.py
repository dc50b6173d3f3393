"""Host NUMA placement helpers (host plumbing for the pinned staging path)."""
import os

from paper_2310_02926_b200 import numa


def test_parse_cpulist():
    assert numa._parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert numa._parse_cpulist("") == []


def test_nodes_and_noop_binding():
    nodes = numa.cpu_nodes()
    for n in nodes:
        assert numa.node_cpus(n)
    assert numa.node_cpus(10_000) == []
    assert numa.bind_to_node(10_000) is False
    before = os.sched_getaffinity(0)
    # no GPU here: the node is unknown, so binding is a no-op
    if len(nodes) < 2:
        assert numa.bind_to_gpu(0) == -1
        assert os.sched_getaffinity(0) == before
