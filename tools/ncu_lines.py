"""Aggregate ncu source-page warp-stall samples by CUDA source line."""
import collections, csv, subprocess, sys

def lines(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    agg = collections.defaultdict(int); src = {}; tot = 0
    cur_file = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]; continue
        if len(r) < 5 or r[0] in ("Line No", "Function Name"):
            continue
        try:
            ln, s = int(r[0]), int(r[4] or 0)
        except ValueError:
            continue
        key = (cur_file, ln)
        agg[key] += s; src[key] = r[1]; tot += s
    print(f"{rep}: {tot} samples")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{v:7d} {100*v/max(tot,1):5.1f}%  {k[0]}:{k[1]:<4}  {src[k].strip()[:90]}")

if __name__ == "__main__":
    lines(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
