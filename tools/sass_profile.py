"""Per-function / hot-window summary of an ncu SASS source page.

ncu -i rep --page source --csv --print-source sass > page.csv
python tools/sass_profile.py page.csv [window]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    h, data = rows[1], rows[2:]
    ix = {k: i for i, k in enumerate(h)}
    S, E, T = (ix['Warp Stall Sampling (All Samples)'], ix['Instructions Executed'],
               ix['Thread Instructions Executed'])
    base = int(data[0][0], 16)
    tot_s = sum(int(r[S]) for r in data) or 1
    tot_e = sum(int(r[E]) for r in data) or 1
    # functions: the kernel from 0, then every CALL target
    starts = {0: "kernel"}
    for r in data:
        t = r[1].strip()
        if "CALL.REL" in t:
            tgt = (int(t.split()[-1], 16) - base) // 16
            starts.setdefault(tgt, f"fn@{tgt}")
    bounds = sorted(starts)
    reasons = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
    print(f"total: {tot_e/1e9:.2f} G warp-inst, {tot_s} stall samples")
    for j, a in enumerate(bounds):
        b = bounds[j + 1] if j + 1 < len(bounds) else len(data)
        seg = data[a:b]
        s = sum(int(r[S]) for r in seg); e = sum(int(r[E]) for r in seg)
        t = sum(int(r[T]) for r in seg)
        mix = collections.Counter()
        for r in seg:
            op = r[1].strip().split()
            op = op[1] if op[0].startswith('@') else op[0]
            mix[op.split('.')[0]] += int(r[E])
        st = collections.Counter({k: sum(int(r[ix[k]] or 0) for r in seg) for k in reasons})
        print(f"{starts[a]:10s} [{a:5d},{b:5d}) stall {100*s/tot_s:5.1f}% inst {100*e/tot_e:5.1f}% "
              f"thr/warp {t/max(e,1):5.1f}")
        if e / tot_e > 0.02:
            print("    ops:", ", ".join(f"{k} {100*v/max(e,1):.0f}" for k, v in mix.most_common(12)))
            print("    stalls:", ", ".join(f"{k[6:]} {100*v/max(s,1):.0f}" for k, v in st.most_common(6)))
    print("hot windows:")
    for a in range(0, len(data), W):
        seg = data[a:a + W]
        s = sum(int(r[S]) for r in seg); e = sum(int(r[E]) for r in seg)
        t = sum(int(r[T]) for r in seg)
        if s / tot_s > 0.015:
            print(f"  {a:5d} stall {100*s/tot_s:5.1f}% inst {e/1e6:9.1f}M thr/warp {t/max(e,1):5.1f}")


if __name__ == "__main__":
    main()
