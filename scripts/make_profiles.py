"""Summarise one gpurun_out/<tag>/ capture into profiles/ (tracked):

    python scripts/make_profiles.py gpurun_out/<tag> <round-tag>

Inputs (see scripts/gpu_session.sh): launches.csv (ncu launch list of
`bench.py --steps 3 --warmup 3`), bench_solve.ncu-rep (ncu --set full of one
bench solve launch), solve.ncu-rep (ncu --set full of a 20-iteration solve,
with source correlation). Outputs: <round>_launches.csv / _launch_shares.txt,
<round>_ncu_bench_solve.txt, <round>_ncu_solve_lines.txt, <round>_ncu_traffic.json.
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO / "scripts"))


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def fnum(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main(src, tag):
    src = Path(src)
    prof = REPO / "profiles"
    prof.mkdir(exist_ok=True)
    # launch list
    lf = src / "launches.csv"
    if lf.exists():
        lines = [l for l in lf.read_text().splitlines() if l.startswith('"')]
        rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
        out = prof / f"{tag}_launches.csv"
        with out.open("w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["id", "kernel", "grid", "block", "ns"])
            for r in rows:
                w.writerow([r["ID"], r["Kernel Name"][:90], r["Grid Size"], r["Block Size"], r["Metric Value"]])
        tot = collections.Counter(); cnt = collections.Counter()
        for r in rows:
            k = r["Kernel Name"].split("(")[0][:70]
            tot[k] += fnum(r["Metric Value"]) or 0
            cnt[k] += 1
        ours = {k: v for k, v in tot.items() if "pm::" in k or "solve_kernel" in k or "psum" in k or "escale" in k}
        s = sum(ours.values()) or 1
        with (prof / f"{tag}_launch_shares.txt").open("w") as f:
            f.write("ncu launch list of `python bench.py --steps 3 --warmup 3 --no-cpu-baseline`\n")
            f.write("(gpu__time_duration.sum, --clock-control none; cold-cache, serialised: compare shares)\n\n")
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
                share = f"{v / s * 100:6.2f}% of our kernels" if k in ours else "   (harness / torch)"
                f.write(f"{cnt[k]:4d} launches  {v / 1e3:10.1f} us total  {share}  {k}\n")
    # full capture of the bench solve launch -> traffic
    bf = src / "bench_solve.ncu-rep"
    if bf.exists():
        rows, units = raw(bf)
        d = rows[0]
        rd, wr = fnum(d["dram__bytes_read.sum"]), fnum(d["dram__bytes_write.sum"])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units["dram__bytes_read.sum"], 1)
        wr *= scale.get(units["dram__bytes_write.sum"], 1)
        dur = fnum(d["gpu__time_duration.sum"]) * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(
            units["gpu__time_duration.sum"], 1)
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
                "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
        with (prof / f"{tag}_ncu_bench_solve.txt").open("w") as f:
            f.write(f"ncu --set full of one bench.py solve launch (1024^2 fp32, 100 GS iterations, L2 flushed before)\n")
            f.write(f"kernel: {d['Kernel Name']}\n")
            for k in keys:
                if k in d:
                    f.write(f"  {k:70s} {d[k]} {units.get(k, '')}\n")
        json.dump({"kernel": d["Kernel Name"], "dram_bytes_read": rd, "dram_bytes_write": wr,
                   "dram_bytes_per_launch": rd + wr, "ncu_duration_ns": dur,
                   "algorithmic_bytes_per_launch": 40 * 1024 * 1024 * 100,
                   "note": "one launch = the whole 100-iteration solve of one 1024^2 fp32 mask; the field is L2-resident, "
                           "so DRAM traffic is the cold first touch plus write-back, far below the algorithmic bytes"},
                  (prof / f"{tag}_ncu_traffic.json").open("w"), indent=1)
    sf = src / "solve.ncu-rep"
    if not sf.exists():
        sf = src / "solve_full.ncu-rep"
    if sf.exists():
        from ncu_lines import main as lines_main
        import contextlib
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            lines_main(str(sf), 40)
        summ = subprocess.run([sys.executable, str(REPO / "scripts" / "ncu_summary.py"), str(sf), "2"],
                              capture_output=True, text=True).stdout
        (prof / f"{tag}_ncu_solve_lines.txt").write_text(
            "ncu --set full --import-source on of a 100-iteration 1024^2 fp32 solve (scripts/prof_solve.py 1024 single 100)\n\n"
            + summ + "\nwarp-stall samples by source line (scripts/ncu_lines.py):\n" + buf.getvalue())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
