"""DRAM traffic per launch of the step's expert GEMMs from an `ncu --set full` capture
(`ncu -i <rep> --page raw --csv > raw.csv`): the wgrad GEMMs with the fused AdamW epilogue
(EPI = 4) and the forward / dgrad GEMMs, averaged per launch -- the `traffic` field of
bench.py's rooflines.  usage: python tools/gemm_traffic.py raw.csv "<workload>" <n_gpus> > json"""
import csv
import json
import sys

path, workload, n_gpus = sys.argv[1], sys.argv[2], int(sys.argv[3])
r = list(csv.reader(open(path)))
h, u, rows = r[0], r[1], r[2:]


def col(name):
    return [i for i, x in enumerate(h) if x == name or x.endswith("." + name)][-1]


scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
kn, rd, wr, tm = col("Kernel Name"), col("dram__bytes_read.sum"), col("dram__bytes_write.sum"), \
    col("gpu__time_duration.sum")
wg, tc = [], []
for row in rows:
    nm = row[kn]
    if "grouped_gemm_kernel" not in nm:
        continue
    b = float(row[rd].replace(",", "")) * scale[u[rd]] + float(row[wr].replace(",", "")) * scale[u[wr]]
    targs = nm.split("grouped_gemm_kernel<", 1)[1].split(">", 1)[0].split(",")
    (wg if targs[2].strip() == "4" else tc).append(b)
print(json.dumps({"workload": workload, "n_gpus": n_gpus,
                  "wgrad_per_launch": sum(wg) / len(wg) if wg else None,
                  "tc_per_launch": sum(tc) / len(tc) if tc else None,
                  "launches": {"wgrad_adam": len(wg), "fwd_dgrad": len(tc)},
                  "source": "ncu --set full (cold cache, serialised replays): dram__bytes_read.sum + "
                            "dram__bytes_write.sum per launch"}))
