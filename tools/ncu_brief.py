"""Brief ncu report reader: headline metrics per kernel and the hottest SASS basic blocks
(runs of equal execution counts). python tools/ncu_brief.py REPORT [kernel-regex] [nblocks]"""
import csv
import io
import re
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Achieved Occupancy', 'Registers Per Thread', 'Compute (SM) Throughput',
        'Executed Ipc Active', 'L2 Hit Rate', 'Mem Busy', 'Max Bandwidth', 'Issue Slots Busy', 'Grid Size',
        'Block Size', 'Dynamic Shared Memory Per Block', 'Block Limit Shared Mem', 'Block Limit Registers']


def main():
    rep = sys.argv[1]
    kre = re.compile(sys.argv[2]) if len(sys.argv) > 2 else re.compile('.')
    nb = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
    seen = set()
    for r in rows[1:]:
        k = (r[ki][:50], r[mi])
        if kre.search(r[ki]) and r[mi] in WANT and k not in seen:
            seen.add(k)
            print(f'{r[ki][:50]:50s} {r[mi]:32s} {r[vi]} {r[ui]}')
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kern, hdr, ds = None, None, {}
    for r in rows:
        if r and r[0] == 'Kernel Name':
            kern = r[1]
            continue
        if r and r[0] == 'Address':
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and kern and kre.search(kern):
            ds.setdefault(kern, []).append(dict(zip(hdr, r)))
    for k, d in ds.items():
        blocks, cur = [], None
        for i, x in enumerate(d):
            n = int(x['Instructions Executed'] or 0)
            s = int(x.get('Warp Stall Sampling (All Samples)') or 0)
            if cur and cur[1] == n:
                cur[2] += 1
                cur[3].append(x['Source'].strip()[:48])
                cur[4] += s
            else:
                cur = [i, n, 1, [x['Source'].strip()[:48]], s]
                blocks.append(cur)
        tot = sum(b[1] * b[2] for b in blocks) or 1
        stot = sum(b[4] for b in blocks) or 1
        print(f'\n{k[:90]}: {tot} warp instructions, {len(d)} SASS')
        for b in sorted(sorted(blocks, key=lambda b: -b[1] * b[2])[:nb]):
            print(f'  @{b[0]:5d} len {b[2]:4d} x{b[1]:>9d} = {100 * b[1] * b[2] / tot:5.1f}% instr, '
                  f'{100 * b[4] / stot:5.1f}% stalls | {" | ".join(b[3][:2])} ... {b[3][-1]}')
        break


if __name__ == '__main__':
    main()
