"""Per-source-line executed instructions / stall samples of the first kernel
in each of two ncu reports, and the lines whose counts differ most."""
import csv, io, subprocess, sys, collections

def lines(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, seen_fn, res = None, 0, collections.Counter()
    samp = collections.Counter()
    text = {}
    for r in rows:
        if r and r[0] == 'Function Name':
            seen_fn += 1
        if seen_fn > 1 and r and r[0] == 'Function Name':
            pass
        if r and r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if len(r) > 8 and r[0] not in ('', 'Line No'):
            try:
                key = (cur, int(r[0]))
            except ValueError:
                continue
            ie = r[5] if False else None
            text[key] = r[1][:80]
            try:
                res[key] += int(r[7]) if r[7] not in ('-', '') else 0
            except ValueError:
                pass
            try:
                samp[key] += int(r[6]) if r[6] not in ('-', '') else 0
            except ValueError:
                pass
    return res, samp, text

if __name__ == '__main__':
    a, sa, ta = lines(sys.argv[1])
    b, sb, tb = lines(sys.argv[2])
    print('total inst', sum(a.values()), sum(b.values()))
    keys = set(a) | set(b)
    d = sorted(keys, key=lambda k: -abs(b[k] - a[k]))
    for k in d[:40]:
        print(k, a[k], b[k], b[k] - a[k], sa[k], sb[k], (ta.get(k) or tb.get(k)))
