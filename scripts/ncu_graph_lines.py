import csv, re, sys, collections
rep, kid, func_pat = sys.argv[1], sys.argv[2], sys.argv[3]
import subprocess
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
blocks, cur = [], None
for ln in out.split('\n'):
    if ln.startswith('"Kernel Name"'):
        cur = []; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
rows = list(csv.reader(blocks[int(kid)])); hdr = rows[0]
ai, ie, si = hdr.index('Address'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
recs = [(int(r[ai], 16), float(r[ie] or 0), float(r[si] or 0), r[1]) for r in rows[1:] if len(r) >= len(hdr)]
base = min(a for a, *_ in recs)
srcfile = open(sys.argv[4] if len(sys.argv) > 4 else '/root/repo/paper_0910_5435_b200/csrc/wgraph.cu').read().split('\n')
dis = open(sys.argv[5] if len(sys.argv) > 5 else '/tmp/dis/wgraph.dis').read().split('\n')
off2line, cur_line, active = {}, None, False
for d in dis:
    if d.startswith('.text.'):
        active = func_pat in d
        continue
    if not active: continue
    m = re.search(r'line (\d+)', d)
    if '//## File' in d and m:
        cur_line = int(m.group(1)) if 'wgraph.cu' in d else -1
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', d)
    if m2: off2line[int(m2.group(1), 16)] = cur_line
agg = collections.defaultdict(lambda: [0.0, 0.0])
ops = collections.defaultdict(lambda: [0.0, 0.0])
for a, n, s, sass in recs:
    ln = off2line.get(a - base)
    agg[ln][0] += n; agg[ln][1] += s
    op = sass.strip().split()[0] if not sass.strip().startswith('@') else sass.strip().split()[1]
    op = op.split('.')[0]
    ops[op][0] += n; ops[op][1] += s
ti = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print('total instr %.4g samples %d' % (ti, ts))
for ln, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:38]:
    txt = srcfile[ln - 1].strip()[:90] if ln and ln > 0 else '?'
    print('%5s  instr %5.1f%%  stall %5.1f%%  %s' % (ln, 100 * n / ti, 100 * s / ts, txt))
print('--- by opcode')
for op, (n, s) in sorted(ops.items(), key=lambda x: -x[1][0])[:24]:
    print('%10s instr %5.1f%% stall %5.1f%%' % (op, 100*n/ti, 100*s/ts))
