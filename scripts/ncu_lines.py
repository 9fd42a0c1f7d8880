"""Per-source-line warp-stall samples of an ncu report (needs -lineinfo):
    python scripts/ncu_lines.py report.ncu-rep [top] [kernel-substring]"""
import csv, subprocess, sys, collections

def main(rep, top=30, kfilter=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg = collections.Counter(); reasons = collections.defaultdict(collections.Counter); text = {}
    cur_file = cur_fn = None; hdr = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]; continue
        if len(r) == 2 and r[0] == "Function Name":
            cur_fn = r[1]; continue
        if r and r[0] == "Line No":
            hdr = r; continue
        if not hdr or len(r) != len(hdr) or not r[0]:
            continue
        if kfilter and (not cur_fn or kfilter not in cur_fn):
            continue
        d = dict(zip(hdr[4:], r[4:]))
        try:
            s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        except ValueError:
            continue
        key = (cur_file, int(r[0]))
        agg[key] += s
        text[key] = r[1].strip()[:80]
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    reasons[key][k[6:]] += float(v)
                except ValueError:
                    pass
    tot = sum(agg.values()) or 1
    for key, v in agg.most_common(top):
        rs = ", ".join(f"{k}={x/v*100:.0f}%" for k, x in reasons[key].most_common(3) if x)
        print(f"{v/tot*100:5.1f}% {key[0]}:{key[1]:<5d} {text[key]:80s} [{rs}]")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else None)
