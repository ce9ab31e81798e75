"""Thread-instructions and stall samples per CUDA source line of one kernel
in an ncu report (SASS addresses mapped with nvdisasm --print-line-info)."""
import collections
import csv
import re
import subprocess
import sys

rep, fn, sass, src_file = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ai, ie = h.index('Address'), h.index('Thread Instructions Executed')
st = h.index('Warp Stall Sampling (All Samples)')
data = {}
for r in rows[2:]:
    try:
        data[int(r[ai], 16)] = (float(r[ie]), float(r[st]))
    except (ValueError, IndexError):
        pass
base = min(data)
txt = open(sass).read()
f = [f for f in re.split(r'\n\s*\.text\.', txt) if fn in f.split('\n', 1)[0]][0]
cur, a2l = None, {}
for line in f.split('\n'):
    m = re.search(r'//## File ".*?", line (\d+)', line)
    if m:
        cur = int(m.group(1))
    m = re.search(r'/\*([0-9a-f]{4,})\*/', line)
    if m:
        a2l[int(m.group(1), 16)] = cur
inst, stall = collections.Counter(), collections.Counter()
for a, (i, s) in data.items():
    inst[a2l.get(a - base)] += i
    stall[a2l.get(a - base)] += s
ti, ts = sum(inst.values()), sum(stall.values())
srcl = open(src_file).read().split('\n')
print("total thread instructions", ti)
for k, v in inst.most_common(top):
    print(f"{v / ti * 100:5.1f}% inst {stall[k] / ts * 100:5.1f}% stall L{k} "
          f"{srcl[k - 1].strip()[:90] if k else ''}")
