"""Summarise one `ncu --metrics ... --csv` capture of a hot kernel (tools/gpu_ncu_metrics.sh)
into the derived quantities SURVEY §8(d) asks for: DRAM bytes vs algorithmic bytes, thread
instructions and shared atomics per input byte, atomic bank conflicts, lane-atomics per
SM-clock, issue utilisation and the stall breakdown. Prints one JSON object.

    python tools/ncu_summarize.py counters.csv NAME FRAMES CFG OP [BINS] [WxH] [GIT_SHA]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scn_synth  # noqa: E402

SMS = 148


def read(path):
    vals, kernel = {}, None
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        kernel = row.get("Kernel Name", kernel)
        v = row["Metric Value"].replace(",", "")
        try:
            vals[row["Metric Name"]] = float(v)
        except ValueError:
            vals[row["Metric Name"]] = v
    return vals, kernel


def main():
    path, name, frames, cfg, op = sys.argv[1:6]
    frames = int(frames)
    v, kernel = read(path)
    wl = scn_synth.WORKLOADS[cfg]
    import dataclasses
    if len(sys.argv) > 6 and int(sys.argv[6]):
        wl = dataclasses.replace(wl, bins=int(sys.argv[6]))
    if len(sys.argv) > 7 and sys.argv[7]:
        w, h = (int(x) for x in sys.argv[7].lower().split("x"))
        wl = dataclasses.replace(wl, width=w, height=h)
    sha = sys.argv[8] if len(sys.argv) > 8 else None
    F = wl.frame_bytes
    in_bytes = frames * F
    dsb = frames * (wl.height // 2) * (wl.width // 2) * 3
    alg = in_bytes + (dsb if op != "hist" else 0) + (frames * 3 * wl.bins * 4 if op != "ds" else 0)
    t = v["gpu__time_duration.sum"] * 1e-9 if v.get("gpu__time_duration.sum") else None  # ns
    rd, wr = v.get("dram__bytes_read.sum", 0.0), v.get("dram__bytes_write.sum", 0.0)
    cyc = v.get("sm__cycles_elapsed.avg")
    atom = v.get("smsp__inst_executed_op_shared_atom.sum", 0.0)
    out = {
        "kernel": kernel, "capture": os.path.basename(path), "config": cfg, "op": op, "frames": frames,
        "bins": wl.bins, "width": wl.width, "height": wl.height, "git_sha": sha,
        "frame_bytes": F, "algorithmic_bytes": alg,
        "dram_read_bytes": rd, "dram_write_bytes": wr,
        "dram_over_algorithmic": (rd + wr) / alg,
        "gpu_time_ms_under_ncu": t * 1e3 if t else None,
        "dram_GBps_under_ncu": (rd + wr) / t / 1e9 if t else None,
        "dram_pct_of_peak": v.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_clock_mhz": v.get("sm__cycles_elapsed.avg.per_second", 0) / 1e6 if isinstance(
            v.get("sm__cycles_elapsed.avg.per_second"), float) else None,
        "issue_active_pct": v.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": v.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "thread_instr_per_input_byte": v.get("smsp__inst_executed.sum", 0) * 32 / in_bytes,
        "warp_instr_alu_per_input_byte": v.get("sm__inst_executed_pipe_alu.sum", 0) * 32 / in_bytes,
        "warp_instr_fma_per_input_byte": v.get("sm__inst_executed_pipe_fma.sum", 0) * 32 / in_bytes,
        "shared_atom_lane_ops_per_input_byte": atom * 32 / in_bytes,
        "shared_atom_wavefronts": v.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"),
        "shared_atom_bank_conflicts": v.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum"),
        "shared_atom_lane_ops_per_sm_clk": atom * 32 / (cyc * SMS) if cyc else None,
        "lds_per_input_byte": v.get("smsp__inst_executed_op_shared_ld.sum", 0) * 32 / in_bytes,
        "sts_warp_instr": v.get("smsp__inst_executed_op_shared_st.sum"),
        "stg_warp_instr": v.get("smsp__inst_executed_op_global_st.sum"),
        "red_global_warp_instr": v.get("smsp__inst_executed_op_global_red.sum"),
        "tma_warp_instr": v.get("sm__inst_executed_pipe_tma.sum"),
        "l2_tex_read_hit_sectors": v.get("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum"),
        "stall_cycles_per_issued_instr": {k.split("stalled_")[1].replace(".ratio", ""): val for k, val in v.items()
                                          if "issue_stalled" in k},
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
