"""SASS opcode mix (executed warp instructions) per kernel of an ncu report:
    python tools/ncu_opmix.py rep.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    kern, hist, hdr = None, None, None
    res = []
    for r in csv.reader(out.splitlines()):
        if r and r[0] == 'Kernel Name':
            if hist:
                res.append((kern, hist))
            kern, hist = r[1], collections.Counter()
            continue
        if r and r[0] == 'Address':
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and hist is not None:
            try:
                n = float(r[5] or 0)
            except ValueError:
                continue
            op = r[1].strip().split()
            if not op:
                continue
            o = op[0]
            if o.startswith('@'):
                o = op[1] if len(op) > 1 else o
            hist[o.split('.')[0]] += n
    if hist:
        res.append((kern, hist))
    for k, h in res:
        tot = sum(h.values())
        print('=====', k[:100], f'total {tot:.4g}')
        for o, n in h.most_common(top):
            print(f'  {o:12s} {n:14.4g} {100 * n / tot:5.1f}%')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
