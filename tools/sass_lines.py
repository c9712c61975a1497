"""Join an ncu SASS source page (csv) with nvdisasm line info: per-source-line
instruction counts and stall samples.  Usage:
  python tools/sass_lines.py <ncu-src.csv> <cubin> <kernel-substring> <steps> [topN]"""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, kname):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur = None
    out = {}
    line = None
    infn = False
    for ln in txt.splitlines():
        m = re.match(r'\s*\.text\.(\S+):', ln)
        if m:
            infn = kname in m.group(1)
            continue
        if not infn:
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
        if m:
            line = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
        if m and line:
            out[int(m.group(1), 16)] = line
    return out


def main():
    src, cubin, kname, steps = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    lm = line_map(cubin, kname)
    rows = list(csv.reader(open(src)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ex = collections.Counter()
    st = collections.Counter()
    tot = tst = 0
    base = None
    for d in rows[2:]:
        try:
            addr = int(d[ix["Address"]], 16)
        except ValueError:
            continue
        if base is None:
            base = addr
        addr -= base
        e = int(d[ix["Instructions Executed"]] or 0)
        s = int(d[ix["Warp Stall Sampling (All Samples)"]] or 0)
        key = lm.get(addr, "?")
        ex[key] += e
        st[key] += s
        tot += e
        tst += s
    print(f"total {tot / steps:.1f} warp-inst/step, {len(lm)} mapped addresses")
    for k, v in sorted(ex.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{k:28s} {v / steps:7.1f}/step {100 * v / tot:5.1f}%  stalls {100 * st[k] / max(tst, 1):5.1f}%")


if __name__ == "__main__":
    main()
