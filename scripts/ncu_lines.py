"""Join ncu per-SASS-address counts with nvdisasm line info: instructions and
stall samples per CUDA source line (diagnostics)."""
import csv, re, sys, collections
src_csv, dis_txt, which = sys.argv[1], sys.argv[2], int(sys.argv[3])
srcfile = open('paper_0910_5435_b200/csrc/engine.cu').read().split('\n')
lines = open(src_csv).read().split('\n')
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
rows = list(csv.reader(blocks[which][1:])); hdr = rows[0]
ai, ie, si = hdr.index('Address'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
recs = [(int(r[ai], 16), float(r[ie] or 0), float(r[si] or 0)) for r in rows[1:] if len(r) >= len(hdr)]
base = min(a for a, _, _ in recs)
name = 'TILi0EEELb%dE' % which
dis = open(dis_txt).read().split('\n')
off2line, cur_line, active = {}, None, False
for d in dis:
    if d.startswith('.text.'):
        active = 'ShtPolicy' + name in d
        continue
    if not active:
        continue
    m = re.search(r'line (\d+)', d)
    if '//## File' in d and m:
        cur_line = int(m.group(1))
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', d)
    if m2:
        off2line[int(m2.group(1), 16)] = cur_line
agg = collections.defaultdict(lambda: [0.0, 0.0])
for a, n, s in recs:
    ln = off2line.get(a - base)
    agg[ln][0] += n
    agg[ln][1] += s
ti = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print('total instr %.3g samples %d' % (ti, ts))
for ln, (n, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    txt = srcfile[ln - 1].strip()[:70] if ln else '?'
    print('%5s  instr %5.1f%%  stall %5.1f%%  %s' % (ln, 100 * n / ti, 100 * s / ts, txt))
