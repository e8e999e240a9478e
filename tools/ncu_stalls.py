"""Top warp-stall PCs of an .ncu-rep (SASS source page), with the two largest stall reasons
and a few preceding instructions for context (development tool, runs here without a GPU)."""
import csv
import subprocess
import sys


def main(path, top=20, ctx=3):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[1]
    data = rows[2:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    cols = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
    tot = sum(int(r[si]) for r in data)
    print(f"total samples {tot}")
    order = sorted(range(len(data)), key=lambda i: -int(data[i][si]))[:top]
    for i in order:
        r = data[i]
        st = sorted(((int(r[hdr.index(c)]), c[6:]) for c in cols), reverse=True)[:2]
        print(f"{int(r[si]):6d} {r[0][-5:]} {r[1][:70]:70s} {st}")
        for r2 in data[max(0, i - ctx):i]:
            print(f"{'':6s} {r2[0][-5:]}   {r2[1][:70]}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(a) for a in sys.argv[2:]))
