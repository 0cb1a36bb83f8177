"""Turn one `ncu --set full` capture of a hot kernel (a .ncu-rep, read with --page raw
--csv) into the traffic summary bench.py reads for roofline.traffic:
profiles/ncu_<kernel>[_<tag>]_summary.json with DRAM bytes per frame and the git SHA of
the captured library, so a stale capture is flagged (bench.py compares it with
scn_version()).

    python tools/ncu_traffic.py REP.ncu-rep KERNEL FRAMES FRAME_BYTES GIT_SHA OUT.json "description"
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, kernel, frames, F, sha, out, desc = sys.argv[1:8]
    frames, F = int(frames), int(F)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO("\n".join(ln for ln in txt.splitlines() if ln.startswith('"')))))
    head, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = head.index(name)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "second": 1.0}[u]
        return v * scale

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    t = get("gpu__time_duration.sum")
    d = {"kernel": kernel, "source": f"{rep.split('/')[-1]} (ncu --set full --clock-control none; {desc})",
         "git_sha": sha, "kernel_name": vals[head.index("Kernel Name")], "frame_bytes": F,
         "frames_per_launch": frames, "dram_bytes_read": rd, "dram_bytes_write": wr,
         "dram_bytes_per_frame": (rd + wr) / frames, "gpu_time_ms_under_ncu": t * 1e3}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main()
