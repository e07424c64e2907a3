"""Summarise an ncu --set full capture of the streaming kernels (run here, no GPU):
  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_summary.md profiles/traffic.json [tokens]
Writes a markdown table of the key metrics per kernel and traffic.json (DRAM bytes per launch)
that bench.py reports as roofline.traffic."""
import csv
import io
import json
import subprocess
import sys

rep, md, tj = sys.argv[1], sys.argv[2], sys.argv[3]
tokens = int(sys.argv[4]) if len(sys.argv) > 4 else 10_000_000
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def name_of(k):
    """stream_kernel<HIST, W, WIDEN, UNROLL, CHUNKED, WC> -> the bench's traffic keys."""
    import re
    pm = re.search(r"pipe_kernel<(\d+), \d+>", k)  # pipelined-flush kernel: <WC, UNROLL>
    if pm:
        wc = int(pm.group(1))
        return "hist_chunks" if wc == 0 else "fused" if wc == 1 else f"score_w{wc}"
    mm = re.search(r"stream_kernel<(\w+), (\d+), \d+, \d+(?:, (\w+))?(?:, (\d+))?>", k)
    if not mm:
        return k[:40]
    hist = mm.group(1) in ("true", "1")
    W = int(mm.group(2))
    chunked = (mm.group(3) or "false") in ("true", "1")
    wc = int(mm.group(4) or 0)
    if wc:  # count-contract: the fused step (W=1 tables) or score-only W=2/4
        return "fused" if wc == 1 else f"score_w{wc}"
    if hist and W == 0:
        return "hist_chunks" if chunked else "hist"
    if hist:
        return "fused_gather"
    return "score" if W == 1 else f"score_w{W}_gather"


out, traffic = [], {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    nm = name_of(d.get("Kernel Name", ""))
    vals = {}
    for m in M:
        if m in hdr:
            i = hdr.index(m)
            vals[m] = (r[i], units[i])
    rd = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * SCALE.get(vals["dram__bytes_read.sum"][1], 1)
    wr = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * SCALE.get(vals["dram__bytes_write.sum"][1], 1)
    shw = float(vals["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"][0].replace(",", ""))
    traffic.setdefault(nm, {"tokens": tokens, "dram_bytes_per_launch": rd + wr, "alg_bytes": tokens * 58 * 8,
                            "shared_wavefronts_per_launch": shw})
    out.append((nm, vals, rd + wr))
with open(md, "w") as f:
    f.write(f"# ncu --set full summary ({rep}; R1, {tokens} tokens, Zipf 1.2)\n\n")
    f.write("| kernel | " + " | ".join(m.split("__")[1] if "__" in m else m for m in M) + " | DRAM bytes / alg bytes |\n")
    f.write("|" + "---|" * (len(M) + 2) + "\n")
    for nm, vals, tb in out:
        f.write(f"| {nm} | " + " | ".join(f"{vals[m][0]} {vals[m][1]}" if m in vals else "" for m in M)
                + f" | {tb / (tokens * 58 * 8):.4f} |\n")
json.dump(traffic, open(tj, "w"), indent=1)
print(open(md).read())
