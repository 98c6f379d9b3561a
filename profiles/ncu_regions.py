import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout.splitlines()
rows=list(csv.reader(out))
hdr=rows[1]; data=rows[2:]
isrc=hdr.index('Source'); iex=hdr.index('Instructions Executed'); ist=hdr.index('Warp Stall Sampling (All Samples)')
tot=sum(int(r[iex]) for r in data); totst=sum(int(r[ist]) for r in data)
# classify by opcode
from collections import Counter
ops=Counter(); 
for r in data:
    src=r[isrc].strip()
    op=src.split()[0]
    if op.startswith('@'): op=src.split()[1]
    ops[op.split('.')[0]]+=int(r[iex])
print("total", tot)
for op,c in ops.most_common(25): print(f"{op:12s} {c/tot*100:6.2f}%")
# find traceback start: first TMEM load (LDTM) row
first_tb=None
for i,r in enumerate(data):
    if 'LDTM' in r[isrc] or 'REDUX' in r[isrc]: first_tb=i; break
if first_tb:
    tb=sum(int(r[iex]) for r in data[first_tb-30:]); tbs=sum(int(r[ist]) for r in data[first_tb-30:])
    print("traceback region from row", first_tb-30, f"instr {tb/tot*100:.1f}% stall {tbs/totst*100:.1f}%")
