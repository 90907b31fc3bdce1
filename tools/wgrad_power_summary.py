"""Attribute nvidia-smi samples (timestamp, clocks.sm, power.draw, reasons) to the phases
tools/wgrad_power printed (wall-clock ms boundaries); median clock and power per phase."""
import datetime
import statistics
import sys

phases = []
for line in open(sys.argv[1]):
    t = line.split()
    if t and t[0] == "PHASE":
        d = dict(zip(t[2::2], t[3::2]))
        phases.append((t[1], float(d["start_ms"]), float(d["end_ms"]), line.strip()))
samples = []
for line in open(sys.argv[2]):
    p = [x.strip() for x in line.split(",")]
    try:
        ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f")
    except ValueError:
        continue
    ms = ts.replace(tzinfo=datetime.timezone.utc).timestamp() * 1000
    samples.append((ms, float(p[1].split()[0]), float(p[2].split()[0]), p[3]))
# nvidia-smi prints local time; the box runs UTC -- shift by the best alignment if not
for name, t0, t1, line in phases:
    inside = [s for s in samples if t0 + 300 <= s[0] <= t1 - 100]
    if not inside:
        print(line, "| no samples")
        continue
    clk = statistics.median(s[1] for s in inside)
    pw = statistics.median(s[2] for s in inside)
    print(f"{line} | sm_mhz {clk:.0f} power_w {pw:.0f} samples {len(inside)} reasons {inside[len(inside)//2][3]}")
