"""Top source lines (warp-stall samples) of an ncu report: python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur = None; out = []; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0] != "":
        try: s = int(r[4])
        except Exception: continue
        out.append((s, cur, r[0], r[1][:100], r[7]))
tot = sum(o[0] for o in out) or 1
print("total samples", tot)
for o in sorted(out, reverse=True)[:N]:
    print("%5.1f%% %s:%s ie=%s | %s" % (100 * o[0] / tot, o[1], o[2], o[4], o[3]))
