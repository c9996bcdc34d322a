"""Summarise an ncu --set full report (.ncu-rep) into JSON: per launch duration, DRAM bytes, FP64-pipe and
issue utilisation (read here with `ncu -i ... --page raw --csv`; no GPU needed).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_summary_r01.json [workload]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_per_sm": "sm__warps_active.avg.per_cycle_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "sm_mhz": "sm__cycles_elapsed.avg.per_second",
    # executed FP64 instruction mix (thread-level, predicated on) and the XU pipe (MUFU.RCP64H seeds)
    "dfma_thread_inst": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dadd_thread_inst": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul_thread_inst": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "xu_warp_inst": "sm__inst_executed_pipe_xu.sum",
    "fp64_warp_inst": "sm__inst_executed_pipe_fp64.sum",
}
SCALE = {"dram_read": 1, "dram_write": 1}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    wl = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {"report": rep, "workload": wl, "launches": []}
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        e = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", ""), "id": int(d["ID"])}
        for k, m in KEYS.items():
            v = d.get(m)
            if v in (None, ""):
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            un = u.get(m, "")
            if k.startswith("dram_"):  # normalise to bytes
                x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(un, 1)
            if k == "duration_ms":
                x *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ms": 1, "nsecond": 1e-6}.get(un, 1)
            e[k] = x
        e["dram_bytes"] = e.get("dram_read", 0.0) + e.get("dram_write", 0.0)
        if "dfma_thread_inst" in e:
            e["fp64_thread_inst"] = e["dfma_thread_inst"] + e.get("dadd_thread_inst", 0.0) + e.get("dmul_thread_inst", 0.0)
        res["launches"].append(e)
    json.dump(res, open(out, "w"), indent=1)
    for e in res["launches"]:
        print(e)


if __name__ == "__main__":
    main()
