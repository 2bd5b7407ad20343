"""bench.py's reference arm (CPU): the N > 1 workload through the compiled reference
(Scheduler::step placements + sharded_attention_merge over the shard bounds) on a bounded sample."""
import pytest

from tests import oracle_lib


@pytest.mark.skipif(oracle_lib.reference() is None, reason="oracle/_ref not built")
def test_reference_arm_multi_sample():
    import bench
    val, info = bench.cpu_reference_multi(2, steps=1, warmup=0, token_budget=20_000, threads=2)
    assert val > 0 and info["kind"] == "reference" and not info["same_config"]
    assert "CP histogram [1, 2]" in info["sample"]
