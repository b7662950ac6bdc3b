"""Summarise an ncu report (key raw metrics per kernel) as JSON lines.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/xxx.jsonl
"""
import csv
import json
import re
import subprocess
import sys

KEYS = re.compile(
    r"^(gpu__time_duration.sum|dram__bytes_read.sum|dram__bytes_write.sum|"
    r"gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|lts__t_sector_hit_rate.pct|"
    r"l1tex__t_sector_hit_rate.pct|lts__throughput.avg.pct_of_peak_sustained_elapsed|"
    r"sm__throughput.avg.pct_of_peak_sustained_elapsed|sm__warps_active.avg.pct_of_peak_sustained_active|"
    r"sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active|launch__registers_per_thread|"
    r"launch__grid_size|launch__block_size|smsp__inst_executed.sum|"
    r"smsp__pcsamp_warps_issue_stalled_(long_scoreboard|short_scoreboard|wait|mio_throttle|barrier|"
    r"math_pipe_throttle|not_selected|selected|lg_throttle|membar|sleeping))$")


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        rec = {"kernel": r[ki][:120]}
        for i, name in enumerate(h):
            if KEYS.match(name):
                v = r[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                rec[f"{name} [{units[i]}]"] = v
        print(json.dumps(rec))


if __name__ == "__main__":
    main(sys.argv[1])
