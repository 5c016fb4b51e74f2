"""Write profiles/ncu_step_traffic.json from one `ncu --set full` capture of the
step kernel (the `traffic` figure bench.py reports next to the roofline).

    python tools/ncu_traffic.py gpurun_out/prof_step_TAG.ncu-rep [summary_name]
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__time_duration.sum": "duration_us",
    "smsp__cycles_active.avg.per_second": "sm_clock_ghz",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "simt_threads_per_inst",
}
SCALE = {"dram_bytes_read": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "dram_bytes_write": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "duration_us": {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3},
         "sm_clock_ghz": {"cycle/second": 1e-9, "cycle/nsecond": 1, "cycle/usecond": 1e-3}}


def main():
    rep = sys.argv[1]
    summary = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(rep)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    names, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": vals[names.index("Kernel Name")][:60],
           "config": "65,536 envs, 16 maps, R=32, diversity 0.3 (bench.py default)",
           "source": f"ncu --set full --clock-control none, one launch ({summary})"}
    for m, key in METRICS.items():
        if m not in names:
            continue
        i = names.index(m)
        v = float(vals[i].replace(",", ""))
        v *= SCALE.get(key, {}).get(units[i], 1)
        res[key] = v
    res["traffic_bytes_per_launch"] = res.get("dram_bytes_read", 0) + res.get("dram_bytes_write", 0)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2305_04180_b200.build import source_hash
    res["source_hash"] = source_hash()  # bench.py reports the capture only for this build
    json.dump(res, open("profiles/ncu_step_traffic.json", "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
