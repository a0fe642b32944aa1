"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel shares of one DIP iteration. Usage:
    python profiles/summarize_launches.py launches.csv [launches_per_iter]"""
import collections
import csv
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    return [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if len(r) > vi]


def main():
    data = load(sys.argv[1])
    ours = [(k, v) for k, v in data if "d2ip" in k]
    # one iteration = the launches between two consecutive data-term kernels
    marks = [i for i, (k, _) in enumerate(ours) if "jac_loss_k" in k]
    if len(marks) >= 3:
        ours = ours[marks[-3] + 1:marks[-2] + 1]
    elif len(sys.argv) > 2:
        per = int(sys.argv[2])
        ours = ours[-2 * per:-per] if len(ours) >= 2 * per else ours[-per:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in ours:
        name = k.split("(")[0].replace("void ", "")[:70]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'us':>9} {'share':>6} {'n':>4}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1] / 1e3:9.1f} {100 * v[1] / tot:5.1f}% {v[0]:4d}  {k}")
    print(f"{tot / 1e3:9.1f} us total over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main()
