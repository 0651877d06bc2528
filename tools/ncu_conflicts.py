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


if __name__ == '__main__' and not (len(sys.argv) > 2 and sys.argv[2] == 'totals'):
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)


def wavefront_totals(path):
    """SASS-level totals per shared-memory op class: executed instructions,
    wavefronts, ideal wavefronts and excess.  ncu's
    l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_{ld,st} also counts the
    extra passes a 64/128-bit access needs by construction (an STS.128 warp
    store is 4 wavefronts even when conflict-free); "excess" = wavefronts -
    ideal is the real conflict cost."""
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == 'Address')
    ix = {k: hdr.index(k) for k in ('Source', 'Instructions Executed', 'L1 Wavefronts Shared',
                                      'L1 Wavefronts Shared Ideal', 'L1 Wavefronts Shared Excessive')}
    tot = {}
    for r in rows:
        if len(r) != len(hdr) or r is hdr:
            continue
        op = r[ix['Source']].strip().split(' ')[0]
        if not (op.startswith('LDS') or op.startswith('STS')):
            continue
        try:
            vals = [float(r[ix[k]] or 0) for k in ('Instructions Executed', 'L1 Wavefronts Shared',
                                                   'L1 Wavefronts Shared Ideal', 'L1 Wavefronts Shared Excessive')]
        except ValueError:
            continue
        t = tot.setdefault(op, [0.0] * 4)
        for i, v in enumerate(vals):
            t[i] += v
    print(f'{"op":10s} {"executed":>14s} {"wavefronts":>14s} {"ideal":>14s} {"excess":>12s}')
    for op, (n, w, i, e) in sorted(tot.items()):
        print(f'{op:10s} {n:14.0f} {w:14.0f} {i:14.0f} {e:12.0f}')


if __name__ == '__main__' and len(sys.argv) > 2 and sys.argv[2] == 'totals':
    wavefront_totals(sys.argv[1])
