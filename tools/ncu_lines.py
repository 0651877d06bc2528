"""Top CUDA source lines of the kernels in an ncu report by warp-stall samples
(build with -lineinfo, capture with --import-source on):
    python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    recs, fname, hdr = [], '', None
    for r in csv.reader(out.splitlines()):
        if len(r) == 2 and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0]:
            try:
                s, ie = float(r[4] or 0), float(r[7] or 0)
            except ValueError:
                continue
            recs.append((s, ie, f'{fname}:{r[0]}', r[1].strip()[:100]))
    tot = sum(x[0] for x in recs) or 1
    toti = sum(x[1] for x in recs) or 1
    print(f'total stall samples {tot:.0f}, warp instructions {toti:.4g}')
    for s, ie, loc, src in sorted(recs, reverse=True)[:top]:
        print(f'{100 * s / tot:5.1f}% smp {100 * ie / toti:5.1f}% inst  {loc:22s} {src}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
