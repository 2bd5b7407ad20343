"""Run bench.py's planner scenario once (for an ncu launch list of K6 / K7)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_21100_b200.attention import DcpContext  # noqa: E402

print(bench.planner_device(DcpContext(0)))
