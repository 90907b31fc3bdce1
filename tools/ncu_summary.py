"""Summarise an `ncu --page raw --csv` export: per launch duration, DRAM bytes and GB/s,
tensor-pipe activity and SM clock (used for profiles/r*_ncu_*.md)."""
import csv
import sys


def find(h, suffix):
    hits = [i for i, x in enumerate(h) if x == suffix or x.endswith("." + suffix)]
    return hits[-1] if hits else None


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
                                 "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                                 "dram__throughput.avg.pct_of_peak_sustained_elapsed"]}
    scale = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    out = []
    for row in rows:
        nm = row[c["Kernel Name"]].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        t_us = num(row[c["gpu__time_duration.sum"]]) * scale[u[c["gpu__time_duration.sum"]]]
        rd = num(row[c["dram__bytes_read.sum"]]) * scale[u[c["dram__bytes_read.sum"]]]
        wr = num(row[c["dram__bytes_write.sum"]]) * scale[u[c["dram__bytes_write.sum"]]]
        tp = row[c["sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]]
        out.append((nm, t_us, rd, wr, (rd + wr) / (t_us * 1e-6) / 1e9,
                    num(row[c["sm__cycles_elapsed.avg.per_second"]]), num(tp),
                    num(row[c["dram__throughput.avg.pct_of_peak_sustained_elapsed"]])))
    print("| kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s | dram % peak | tensor pipe % | SM GHz |")
    print("|---|---|---|---|---|---|---|---|")
    for nm, t, rd, wr, gbs, clk, tp, dp in out:
        print(f"| {nm[:60]} | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {gbs:.0f} | {dp:.1f} | "
              f"{tp:.1f} | {clk:.2f} |")
    return out


if __name__ == "__main__":
    main(sys.argv[1])
