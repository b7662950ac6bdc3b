"""One exact mu-EG step line of a BASELINE config (bench.exact_step_line),
for launch lists:  ncu --metrics gpu__time_duration.sum ... python tools/step_cfg.py 5"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

if __name__ == "__main__":
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    print(json.dumps(bench.exact_step_line(cfg, steps=steps, warmup=2)))
