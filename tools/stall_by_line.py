import csv,re,sys,collections,subprocess
rep, fn_pat, cubin = sys.argv[1], sys.argv[2], sys.argv[3]
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(src.splitlines()))
h=rows[1]; ai=h.index('Address'); si=h.index('Warp Stall Sampling (All Samples)'); ii=h.index('Source')
samples={}
for r in rows[2:]:
    if len(r)>si:
        try: samples[int(r[ai],16) if r[ai].startswith('0x') else int(r[ai])]=(float(r[si]), r[ii])
        except: pass
txt=open(cubin).read()
funcs=re.split(r'\n\s*\.text\.',txt)
f=[f for f in funcs if fn_pat in f.split('\n',1)[0]][0]
cur=None; addr2line={}
for l in f.split('\n'):
    m=re.search(r'//## File ".*?", line (\d+)',l)
    if m: cur=int(m.group(1))
    m=re.search(r'/\*([0-9a-f]{4,})\*/',l)
    if m: addr2line[int(m.group(1),16)]=cur
base=min(samples)
byline=collections.Counter()
for a,(s,ins) in samples.items(): byline[addr2line.get(a-base)]+=s
tot=sum(byline.values())
srcl=open(sys.argv[5] if len(sys.argv)>5 else '/root/repo/paper_1407_2074_b200/csrc/render.cu').read().split('\n')
for k,v in byline.most_common(int(sys.argv[4]) if len(sys.argv)>4 else 40):
    print(f"{v/tot*100:5.1f}% L{k} {srcl[k-1].strip()[:100] if k else ''}")
