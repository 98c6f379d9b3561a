import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout.splitlines()
rows=list(csv.reader(out))
hdr=rows[1]; data=rows[2:]
isrc=hdr.index('Source'); iex=hdr.index('Instructions Executed'); ist=hdr.index('Warp Stall Sampling (All Samples)')
tot=sum(int(r[iex]) for r in data); totst=sum(int(r[ist]) for r in data)
print("total warp-instr", tot, "rows", len(data))
blocks=[]; cur=None
for i,r in enumerate(data):
    c=int(r[iex])
    if cur is None or c!=cur[0]:
        cur=[c,i,i,0,0]; blocks.append(cur)
    cur[2]=i; cur[3]+=c; cur[4]+=int(r[ist])
for b in blocks:
    if b[3]/tot>0.004 or b[4]/totst>0.01: print(f"rows {b[1]:5d}-{b[2]:5d} count={b[0]:>10} n={b[2]-b[1]+1:4d} instr%={b[3]/tot*100:6.2f} stall%={b[4]/totst*100:6.2f}  {data[b[1]][isrc].strip()[:50]}")
top=sorted(range(len(data)), key=lambda i:-int(data[i][ist]))[:15]
print("top stall instructions:")
for i in top: print(i, data[i][ist].rjust(6), data[i][isrc].strip()[:70])
