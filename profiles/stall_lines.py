import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 14
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv", "-k", "regex:" + kern, "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
isamp = hdr.index("# Samples"); iex = hdr.index("Instructions Executed")
st = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
agg = [r for r in rows[hi + 1:] if len(r) > isamp and r[2] == "-" and r[0].isdigit()]
tot = sum(int(r[isamp] or 0) for r in agg); tote = sum(int(r[iex] or 0) for r in agg)
print(kern, "samples", tot, "instr", tote)
top = sorted(agg, key=lambda r: -int(r[isamp] or 0))[:top_n]
for r in sorted(top, key=lambda r: int(r[0])):
    sts = sorted(((int(r[i] or 0), h) for h, i in st.items()), reverse=True)[:2]
    print(r[0], "%5.1f%%" % (100 * int(r[isamp]) / tot), "%5.1f%%" % (100 * int(r[iex] or 0) / max(tote, 1)), r[1].strip()[:86], [f"{h[6:]}:{n}" for n, h in sts])
