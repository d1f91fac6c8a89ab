"""Run one C4 (10^6 x 32, depth 8) tree through the bench's scale_c4 (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = ["bench.py"]
import torch
import bench
ctx = {"dev": torch.device("cuda", 0), "world": 1, "rank": 0, "flush": torch.empty(1 << 20, dtype=torch.uint8, device="cuda"), "barrier": lambda: None,
       "stream": torch.cuda.current_stream(), "graphed": True, "max": lambda x: x}
try:
    print(bench.scale_c4(ctx, 1, 1))
except Exception as e:  # noqa: BLE001
    print("ERR", e)
