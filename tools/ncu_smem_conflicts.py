"""Shared-memory excessive wavefronts (bank conflicts) per source line of one kernel in an
ncu report: python tools/ncu_smem_conflicts.py report.ncu-rep <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
cur, hdr, res = None, None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and cur and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            ex = int(d.get("L1 Wavefronts Shared Excessive", "0") or 0)
            tot = int(d.get("L1 Wavefronts Shared", "0") or 0)
        except ValueError:
            continue
        if tot:
            res.append((ex, tot, cur.split("/")[-1], int(r[0]), r[1].strip()[:70]))
E = sum(x[0] for x in res)
T = sum(x[1] for x in res)
print(f"shared wavefronts {T}, excessive {E} ({100.0 * E / max(T, 1):.1f} %)")
for ex, tot, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{ex:>10} / {tot:>10}  {f}:{ln}  {src}")
