"""configs[0] latency (one 7x7 window, T = 49, C = 768) and small-T op #6 plans: prints the bench's
config0_window object plus per-T layer latencies for the shard sizes of the multi-GPU configs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

if __name__ == "__main__":
    print(json.dumps(bench.window_latency(int(sys.argv[1]) if len(sys.argv) > 1 else 50)), flush=True)
