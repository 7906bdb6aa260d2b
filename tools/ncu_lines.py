"""Top source lines by warp-stall samples from an ncu report (source page,
CUDA + SASS interleaved).  usage: python tools/ncu_lines.py <rep> [N]"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, agg = "?", None, []
    for row in rows:
        if len(row) == 2 and row[0] == "File Path":
            fname = row[1].rsplit("/", 1)[-1]
            continue
        if row and row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row or not row[0]:
            continue
        d = dict(zip(hdr, row))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        stalls = {k[6:]: int(v) for k, v in zip(hdr, row) if k.startswith("stall_") and v.isdigit() and int(v) > 0}
        agg.append((s, fname, row[0], row[1].strip()[:90], stalls))
    tot = sum(a[0] for a in agg)
    agg.sort(key=lambda a: -a[0])
    print("total samples", tot)
    for s, f, ln, src, st in agg[:top]:
        top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print("%5d %5.1f%% %s:%s  %s  %s" % (s, 100.0 * s / max(tot, 1), f, ln, src, top3))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
