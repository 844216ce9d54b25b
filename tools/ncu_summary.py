"""Summarise ncu outputs for profiles/:

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of a launch list
    python tools/ncu_summary.py full <report.ncu-rep> [traffic.json] # key metrics per captured kernel

`full` also writes per-kernel DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) to the
optional traffic.json (kernel label -> bytes), which bench.py reports as roofline.traffic.
"""
import collections
import csv
import io
import json
import subprocess
import sys

LABELS = {  # ncu kernel name prefix -> library profiling label
    "window_attn_kernel": "window_attention", "window_attn_ws_kernel": "window_attention",
    "scan_pass1_kernel": "scan_pass1", "scan_pass2_kernel": "scan_pass2", "scan_dt_kernel": "scan_dt",
    "scan_carry_kernel": "scan_carry", "conv_silu_kernel": "conv_silu", "layer_norm_kernel": "layer_norm",
    "pad_qkv_kernel": "pad_qkv", "pad_tables_kernel": "pad_tables",
}


def gemm_labels(names):
    """Library label of each GEMM launch from its neighbours in the step's launch order (layer structure:
    LN -> QKV -> [pad] -> attention -> out-proj [-> LN2 -> fc1 -> fc2]; LN_s -> in_proj -> conv -> x_proj ->
    dt (TF32 GEMM) -> pass1 / carry / pass2 -> out_proj_scan)."""
    out = []
    for i, n in enumerate(names):
        if n != "gemm_bf16_kernel":
            out.append(LABELS.get(n, n))
            continue
        prev = names[i - 1] if i > 0 else ""
        prev_lab = out[-1] if out else ""
        nxt = names[i + 1] if i + 1 < len(names) else ""
        if prev == "conv_silu_kernel":
            out.append("gemm_x_proj")
        elif prev_lab == "gemm_x_proj":
            out.append("scan_dt")
        elif prev == "scan_pass2_kernel":
            out.append("gemm_out_proj_scan")
        elif prev.startswith("window_attn"):
            out.append("gemm_out_proj")
        elif nxt == "conv_silu_kernel":
            out.append("gemm_in_proj")
        elif prev_lab == "gemm_fc1_gelu":
            out.append("gemm_fc2")
        elif nxt == "gemm_bf16_kernel":
            out.append("gemm_fc1_gelu")
        else:
            out.append("gemm_qkv_rope")
    return out


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("pscwin::", "")
    return n.split("<")[0]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) > vi and "::" not in short(r[ki]):  # library kernels only (torch's L2-flush fills excluded)
            agg.setdefault(short(r[ki]), []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | share of GPU time |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot:.3f} |")


UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,  # -> us
        "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}       # -> MB

METRICS = [
    ("gpu__time_duration.sum", "us", None),
    ("dram__bytes_read.sum", "MB rd", None),
    ("dram__bytes_write.sum", "MB wr", None),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %", 1),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU %", 1),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %", 1),
    ("launch__registers_per_thread", "regs", 1),
]


def full(path, traffic_out=None, labels_override=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    print("| kernel | " + " | ".join(m[1] for m in METRICS) + " | top stalls (warps per issue) |")
    print("|---" * (len(METRICS) + 2) + "|")
    traffic = {}
    labels = labels_override or gemm_labels([short(r[ki]) for r in rows[2:]])
    for r, lab in zip(rows[2:], labels):
        vals = []
        for key, _, scale in METRICS:
            try:
                i = hdr.index(key)
                sc = UNIT.get(units[i], 1.0) if scale is None else scale
                vals.append(f"{float(r[i].replace(',', '')) * sc:.2f}")
            except (ValueError, IndexError):
                vals.append("?")
        st = sorted(((float(r[i] or 0), hdr[i][len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                     for i in stall_cols), reverse=True)[:3]
        print(f"| {lab} | " + " | ".join(vals) + " | " + ", ".join(f"{n} {v:.2f}" for v, n in st) + " |")
        try:
            ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            b = 1e6 * (float(r[ir].replace(",", "")) * UNIT.get(units[ir], 1e-6) +
                       float(r[iw].replace(",", "")) * UNIT.get(units[iw], 1e-6))
            traffic.setdefault(lab, b)
        except (ValueError, IndexError):
            pass
    if traffic_out:
        with open(traffic_out, "w") as f:
            json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        # optional 4th argument: comma-separated labels of the captured launches, in order (a -k filtered capture
        # has no neighbouring kernels to infer the GEMM labels from)
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] != "-" else None,
             sys.argv[4].split(",") if len(sys.argv) > 4 else None)
