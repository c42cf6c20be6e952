"""Times the GTN constitutive update at 256^3 (bench.gtn_measurement) -- the command profiled by ncu."""
import json, sys, torch
sys.path.insert(0, ".")
import bench
dev = torch.device("cuda", 0)
print(json.dumps(bench.gtn_measurement(256, dev, 6449.1, reps=int(sys.argv[1]) if len(sys.argv) > 1 else 3)))
