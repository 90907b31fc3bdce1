"""Summarise an `ncu --page raw --csv` export: per launch duration, DRAM bytes and GB/s,
DRAM % of peak, tcgen05 (UTCHMMA bf16) tensor-op utilisation, mma.sync tensor-pipe activity
and SM clock (used for profiles/r*_ncu_*.md).  The tcgen05 figure is
sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off (the older
sm__pipe_tensor_cycles_active counter does not see tcgen05 MMAs)."""
import csv
import sys


def find(h, *suffixes):
    for suffix in suffixes:
        hits = [i for i, x in enumerate(h) if x == suffix or x.endswith("." + suffix)]
        if hits:
            return hits[-1]
    return None


def cell(row, i):
    return row[i] if i is not None else "nan"


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return float("nan")


def main(path):
    r = list(csv.reader(open(path)))
    h, u, rows = r[0], r[1], r[2:]
    c = {k: find(h, k) for k in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                 "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
                                 "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]}
    c["dram_pct"] = find(h, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                         "dram__throughput.avg.pct_of_peak_sustained_elapsed")
    c["utc"] = find(h, "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg."
                       "pct_of_peak_sustained_elapsed")
    scale = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    out = []
    for row in rows:
        nm = row[c["Kernel Name"]].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        t_us = num(row[c["gpu__time_duration.sum"]]) * scale[u[c["gpu__time_duration.sum"]]]
        rd = num(row[c["dram__bytes_read.sum"]]) * scale[u[c["dram__bytes_read.sum"]]]
        wr = num(row[c["dram__bytes_write.sum"]]) * scale[u[c["dram__bytes_write.sum"]]]
        tp = cell(row, c["sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"])
        clk_u = u[c["sm__cycles_elapsed.avg.per_second"]] if c["sm__cycles_elapsed.avg.per_second"] is not None else ""
        clk = num(cell(row, c["sm__cycles_elapsed.avg.per_second"]))
        clk = clk / 1e9 if clk_u in ("cycle/second", "cycle/s", "") and clk > 1e6 else clk
        out.append((nm, t_us, rd, wr, (rd + wr) / (t_us * 1e-6) / 1e9, clk, num(tp),
                    num(cell(row, c["dram_pct"])), num(cell(row, c["utc"]))))
    print("| kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s | dram % peak | tcgen05 bf16 % | mma.sync pipe % | SM GHz |")
    print("|---|---|---|---|---|---|---|---|---|")
    for nm, t, rd, wr, gbs, clk, tp, dp, utc in out:
        print(f"| {nm[:60]} | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {gbs:.0f} | {dp:.1f} | "
              f"{utc:.1f} | {tp:.1f} | {clk:.2f} |")
    return out


if __name__ == "__main__":
    main(sys.argv[1])
