"""Source lines with excess shared-memory wavefronts (bank conflicts) in an ncu report
(build with -lineinfo, capture with --import-source on):
    python tools/ncu_conflicts.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys


def main(path, top=12):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    hdr, fname, rows = None, '', []
    for r in csv.reader(out.splitlines()):
        if len(r) == 2 and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0]:
            i_ex, i_w = hdr.index('L1 Wavefronts Shared Excessive'), hdr.index('L1 Wavefronts Shared')
            try:
                ex, w = float(r[i_ex] or 0), float(r[i_w] or 0)
            except ValueError:
                continue
            if ex > 0:
                rows.append((ex, w, f'{fname}:{r[0]}', r[1].strip()[:90]))
    for ex, w, loc, src in sorted(rows, reverse=True)[:top]:
        print(f'{ex:12.0f} excess of {w:12.0f}  {loc:20s} {src}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
