"""Summarise an ncu --set full report into profiles/: per-kernel duration,
DRAM bytes (the `traffic` of bench.py's roofline), throughput and the top
stall reasons.  Usage: python tools/ncu_summary.py <rep> <tag>"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
NAMES = {"reduce_kernel<wf::<unnamed>::SumI32": "reduce_sum_i32",
         "reduce_kernel<unnamed>::SumI32": "reduce_sum_i32",
         "reduce_kernel<unnamed>::SumF32": "reduce_sum_f32",
         "reduce_kernel<wf::<unnamed>::SumF32": "reduce_sum_f32",
         "scan_i32_kernel": "scan_inclusive_i32", "tile_persistent_kernel<false>": "scan_inclusive_i32",
         "tile_persistent_kernel<(bool)0>": "scan_inclusive_i32",
         "tile_persistent_kernel<(bool)1>": "compact_gt0_i32",
         "tile_persistent_kernel<true>": "compact_gt0_i32",
         "tile_persistent_kernel<0>": "scan_inclusive_i32", "tile_persistent_kernel<1>": "compact_gt0_i32",
         "compact_gt0_kernel": "compact_gt0_i32", "hist256_kernel": "histogram256_u8",
         "tile_tmem_kernel<false>": "scan_inclusive_i32", "tile_tmem_kernel<(bool)0>": "scan_inclusive_i32",
         "tile_tmem_kernel<0>": "scan_inclusive_i32", "tile_tmem_kernel<true>": "compact_gt0_i32",
         "tile_tmem_kernel<(bool)1>": "compact_gt0_i32", "tile_tmem_kernel<1>": "compact_gt0_i32",
         # two template parameters since the fused multi-GPU form: <COMPACT, PX>
         "tile_tmem_kernel<0, ": "scan_inclusive_i32", "tile_tmem_kernel<1, ": "compact_gt0_i32",
         "tile_tmem_kernel<(bool)0, ": "scan_inclusive_i32",
         "tile_tmem_kernel<(bool)1, ": "compact_gt0_i32",
         "warp_partials_kernel<1>": "warp_partials_sum_f32 (reference C1_F32 text)",
         "warp_partials_kernel<true>": "warp_partials_sum_f32 (reference C1_F32 text)",
         "warp_partials_kernel<(bool)1>": "warp_partials_sum_f32 (reference C1_F32 text)",
         "warp_prefix32_vec_kernel": "warp_prefix32_i32 (reference C3_WARP_PREFIX text)"}


def op_name(kernel: str) -> str:
    for k, v in NAMES.items():
        if k in kernel:
            return v
    return kernel[:40]


def main(rep: str, tag: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def g(r, name, scale=1.0):
        v = r[col[name]] if name in col else ""
        try:
            return float(v.replace(",", "")) * scale
        except ValueError:
            return None

    stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    out, traffic = [], {}
    for r in rows[2:]:
        name = op_name(r[col["Kernel Name"]])
        ms = g(r, "gpu__time_duration.sum")
        unit = units[col["gpu__time_duration.sum"]]
        ms = ms / 1e3 if unit == "us" else (ms / 1e6 if unit == "ns" else ms)
        sc = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rd = g(r, "dram__bytes_read.sum", sc.get(units[col["dram__bytes_read.sum"]], 1.0))
        wr = g(r, "dram__bytes_write.sum", sc.get(units[col["dram__bytes_write.sum"]], 1.0))
        stalls = sorted(((g(r, h) or 0.0, h.replace("smsp__average_warps_issue_stalled_", "")
                          .replace("_per_issue_active.ratio", "")) for h in stall_cols),
                        reverse=True)[:4]
        rec = {"op": name, "grid": r[col["launch__grid_size"]],
               "block": r[col["launch__block_size"]], "ms": round(ms, 5),
               "dram_read_bytes": rd, "dram_write_bytes": wr,
               "dram_gbs": round((rd + wr) / (ms * 1e-3) / 1e9, 1) if ms else None,
               "dram_pct_peak": g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
               "regs": g(r, "launch__registers_per_thread"),
               "warps_active_pct": g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
               "top_stalls": [(n, round(v, 2)) for v, n in stalls]}
        out.append(rec)
        traffic[name] = int(rd + wr)
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    (prof / f"{tag}_ncu_full.json").write_text(json.dumps(out, indent=1))
    tj = prof / "ncu_traffic.json"
    cur = json.loads(tj.read_text()) if tj.exists() else {}
    cur.update(traffic)
    tj.write_text(json.dumps(cur, indent=1))
    lines = [f"# ncu --set full summary ({tag})", "",
             "| op | grid x block | ms (ncu, cold) | DRAM read | DRAM write | DRAM GB/s | DRAM % peak | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|"]
    for o in out:
        lines.append(f"| {o['op']} | {o['grid']} x {o['block']} | {o['ms']} | {o['dram_read_bytes']:.4g} | "
                     f"{o['dram_write_bytes']:.4g} | {o['dram_gbs']} | {o['dram_pct_peak']} | "
                     f"{o['regs']} | {', '.join(f'{n} {v}' for n, v in o['top_stalls'])} |")
    (prof / f"{tag}_ncu_full.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
