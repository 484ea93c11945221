"""Per-source-line stall samples of one kernel in an ncu report (needs -lineinfo).
usage: python tools/ncu_hot_lines.py report.ncu-rep <kernel-regex> [top] [launch-skip]"""
import csv, subprocess, sys, io
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, res = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]; continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; continue
    if hdr and cur and len(r) == len(hdr) and r[0].isdigit():
        vals = dict(zip(hdr[2:], r[2:]))  # skip the duplicate 'Source' column pair
        try:
            s = int(r[4] or 0)
        except ValueError:
            continue
        if s:
            stalls = {}
            for k, v in zip(hdr, r):
                if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0:
                    stalls[k[6:]] = int(v)
            res.append((s, cur.split("/")[-1], int(r[0]), r[1].strip()[:64], stalls))
tot = sum(x[0] for x in res)
res.sort(key=lambda x: -x[0])
print(f"total samples {tot}")
for s, f, ln, src, st in res[:top]:
    top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{s/tot*100:5.1f}% {f}:{ln:<4d} {src:64s} {top3}")
