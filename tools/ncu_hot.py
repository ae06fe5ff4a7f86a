"""Top SASS instructions by warp-stall samples from an ncu report
(ncu -i REP --page source --csv), with their dominant stall reason."""
import csv
import subprocess
import sys


def main(rep, kernel_regex, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel_regex}"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    hi = [i for i, r in enumerate(rows) if "# Samples" in r][0]
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[idx["# Samples"]] or 0) for r in data)
    print("total samples", tot, "instructions", len(data))
    order = sorted(range(len(data)), key=lambda k: -int(data[k][idx["# Samples"]] or 0))[:top]
    for k in sorted(order):
        r = data[k]
        s = int(r[idx["# Samples"]] or 0)
        best = max(stalls, key=lambda h: int(r[idx[h]] or 0))
        print(f"{k:5d} {s:6d} {100 * s / max(tot, 1):5.1f}% {best:22s} {r[idx['Source']].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
