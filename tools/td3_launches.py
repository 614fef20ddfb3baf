"""A few replays of the TD3 update-pair graph at a config (for an ncu launch list of one pair).
Usage: python tools/td3_launches.py [cfg1] [pairs]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.set_device(0)
td3, shape, B = bench.build_td3(name, 1, 0, "auto", 100_000)
td3.update_pair(1)
td3.capture_pair()
for _ in range(n):
    td3.replay_pair()
torch.cuda.synchronize()
print("ok")
