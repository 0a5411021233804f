"""Summarise an ncu --set full report (.ncu-rep) into markdown: per-kernel key metrics and
the top source lines by stall samples (needs -lineinfo + --import-source on)."""
import csv, io, subprocess, sys, collections

KEYS = ["Duration", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Avg. Not Predicated Off Threads Per Warp",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, title, nlines=12):
    out = [f"## {title}", "", f"source: `{rep}` (ncu --set full --clock-control none --import-source on)", ""]
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0].replace("void ", ""))
        if r[ix["Metric Name"]] in KEYS:
            per.setdefault(key, {})[r[ix["Metric Name"]]] = f'{r[ix["Metric Value"]]} {r[ix["Metric Unit"]]}'.strip()
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    rh = raw[0]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum"]
    for r in raw[2:]:
        d = dict(zip(rh, r))
        key = (d.get("ID"), d.get("Kernel Name", "").split("(")[0].replace("void ", ""))
        for w in want:
            if w in d and key in per:
                per[key][w] = d[w] + " " + (raw[1][rh.index(w)] if len(raw) > 1 else "")
    for (kid, name), m in per.items():
        out.append(f"### launch {kid}: `{name}`")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k in KEYS + want:
            if k in m:
                out.append(f"| {k} | {m[k]} |")
        out.append("")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
