"""Extract one verify step (k_prep .. k_set_len, the last complete one) from an ncu launch log
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L ...`) and print the
per-kernel share; writes the step's launches as idx,kernel,grid,block,duration_us.
Usage: python tools/launch_list.py L out.csv "title" """
import collections
import csv
import sys


def main():
    src, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(open(src)) if len(r) > 10 and r[0] != "ID"]
    hdr = next(r for r in csv.reader(open(src)) if r and r[0] == "ID")
    ix = {n: i for i, n in enumerate(hdr)}
    seq = []
    for r in rows:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("::")[-1]
        if "<" in r[ix["Kernel Name"]]:
            base = r[ix["Kernel Name"]].replace("void ", "")
            name = base.split("(")[0].split("::")[-1]
        val = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = val / 1000.0 if unit in ("ns", "nsecond") else (val * 1000.0 if unit in ("ms", "msecond") else val)
        seq.append((name, r[ix["Grid Size"]], r[ix["Block Size"]], us))
    ends = [i for i, s in enumerate(seq) if s[0].startswith("k_set_len")]
    starts = [i for i, s in enumerate(seq) if s[0].startswith("k_prep")]
    e = ends[-1]
    b = max(i for i in starts if i < e)
    step = seq[b:e + 1]
    with open(out, "w") as f:
        f.write(f"# {title}\n")
        f.write("idx,kernel,grid,block,duration_us\n")
        for i, (n, g, bl, us) in enumerate(step):
            f.write(f'{i},{n},"{g}","{bl}",{us:.3f}\n')
    agg = collections.defaultdict(list)
    for n, _, _, us in step:
        agg[n].append(us)
    tot = sum(sum(v) for v in agg.values())
    print(f"{len(step)} launches, {tot / 1000:.3f} ms")
    for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{n:36s} {100 * sum(v) / tot:5.1f}%  n={len(v):4d} mean={sum(v) / len(v):8.2f} us")


if __name__ == "__main__":
    main()
