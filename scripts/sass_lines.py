"""Per-source-line totals of an ncu SASS source page (instructions executed,
warp-stall samples), mapped through nvdisasm -g line info of the object that
holds the kernel. Usage: sass_lines.py REPORT KERNEL_REGEX OBJ MANGLED_NAME"""
import csv, io, re, subprocess, sys, collections, os, tempfile
rep, kre, obj, mangled = sys.argv[1:5]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name-base", "demangled", "--kernel-name",
                      "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
seen = set(); sass = []
for r in data:
    if r and r[0] == "Kernel Name":
        break
    if r[0] in seen: continue
    seen.add(r[0]); sass.append(r)
base = int(sass[0][0], 16)
ie = hdr.index("Instructions Executed"); iw = hdr.index("Warp Stall Sampling (All Samples)")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
full = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
parts = re.split(r"\n\s*\.text\.(\S+):", full)
dis = next(parts[i + 1] for i in range(1, len(parts), 2) if parts[i] == mangled)
line_of = {}
cur = None
for l in dis.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (os.path.basename(m.group(1)), int(m.group(2)))
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur: line_of[int(m.group(1), 16)] = cur
tot_i = collections.Counter(); tot_w = collections.Counter()
for r in sass:
    off = int(r[0], 16) - base
    key = line_of.get(off, ("?", 0))
    tot_i[key] += float(r[ie] or 0); tot_w[key] += float(r[iw] or 0)
ti = sum(tot_i.values()); tw = sum(tot_w.values())
print(f"instructions {ti:.0f}  stall samples {tw:.0f}")
for k, v in sorted(tot_i.items(), key=lambda x: -x[1])[:35]:
    print(f"{k[0]:>18}:{k[1]:<5} instr {100*v/ti:5.1f}%  stalls {100*tot_w[k]/max(tw,1):5.1f}%")
print("-- by stall samples")
for k, v in sorted(tot_w.items(), key=lambda x: -x[1])[:20]:
    print(f"{k[0]:>18}:{k[1]:<5} instr {100*tot_i[k]/ti:5.1f}%  stalls {100*v/max(tw,1):5.1f}%")
