"""Stall reasons of an ncu SASS source page aggregated per innermost SASS loop
(= per FFT stage of the warp-line kernel). Usage: stall_by_loop.py REPORT OBJ MANGLED"""
import csv, io, re, subprocess, sys, os, tempfile, collections
rep, obj, mangled = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name": break
    data.append(r)
base = int(data[0][0], 16)
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = {h: hdr.index(h) for h in cols}
ie = hdr.index("Instructions Executed")
per_off = {}
for r in data:
    off = int(r[0], 16) - base
    per_off[off] = (float(r[ie] or 0), {h: float(r[ci[h]] or 0) for h in cols}, r[1])
# loops from the disassembly
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
full = subprocess.run(["nvdisasm", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
parts = re.split(r"\n\s*\.text\.(\S+):", full)
dis = next(parts[i + 1] for i in range(1, len(parts), 2) if parts[i] == mangled)
instrs, labels = [], {}
for l in dis.split("\n"):
    m = re.match(r"\s*\.L_x_(\d+):", l)
    if m: labels[int(m.group(1))] = len(instrs)
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m: instrs.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for k, (a, t) in enumerate(instrs):
    m = re.search(r"BRA\s+`\(\.L_x_(\d+)\)", t)
    if m and int(m.group(1)) in labels and labels[int(m.group(1))] < k:
        s = labels[int(m.group(1))]
        if k - s >= 60: loops.append((instrs[s][0], a))
loops = [l for l in loops if not any(o[0] <= l[0] and l[1] <= o[1] and o != l and (o[1] - o[0]) < 40000 for o in loops)]
tot_samples = sum(sum(v[1].values()) for v in per_off.values())
print(f"total stall samples {tot_samples:.0f}")
covered = 0
for lo, hi in sorted(set(loops)):
    if hi - lo > 40000: continue
    ins = sum(v[0] for o, v in per_off.items() if lo <= o <= hi)
    st = collections.Counter()
    for o, v in per_off.items():
        if lo <= o <= hi:
            for h, x in v[1].items(): st[h] += x
    tot = sum(st.values()); covered += tot
    kinds = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", per_off[o][2]).split()[0].split(".")[0] for o in per_off if lo <= o <= hi)
    sig = ",".join(k for k, _ in kinds.most_common(4))
    print(f"{lo:#7x}-{hi:#7x} [{sig}] instr {ins/1e6:7.2f}M  samples {100*tot/tot_samples:5.1f}%  " +
          " ".join(f"{h[6:]}:{100*x/max(tot,1):.0f}" for h, x in st.most_common(6)))
print(f"outside these loops: {100*(tot_samples-covered)/tot_samples:.1f}% of samples")
inloop = set()
for lo, hi in sorted(set(loops)):
    if hi - lo > 40000: continue
    for o in per_off:
        if lo <= o <= hi: inloop.add(o)
st = collections.Counter(); top = []
for o, v in per_off.items():
    if o in inloop: continue
    for h, x in v[1].items(): st[h] += x
    top.append((sum(v[1].values()), o, v[2], max(v[1].items(), key=lambda kv: kv[1])[0]))
tot = sum(st.values())
print("outside loops:", " ".join(f"{h[6:]}:{100*x/max(tot,1):.0f}" for h, x in st.most_common(8)))
for smp, o, src, why in sorted(top, reverse=True)[:12]:
    print(f"   {o:#7x} {100*smp/tot_samples:5.1f}% {why[6:]:14s} {src[:70]}")
