"""Sum per-line instruction counts (output of tools/sass_lines.py) into named line ranges.
  python tools/sass_lines.py ... 2000 | python tools/region_sum.py <file-substring> name:start name:start ..."""
import re
import sys

fsub = sys.argv[1]
marks = sorted((int(a.split(":")[1]), a.split(":")[0]) for a in sys.argv[2:])
tot, st = {}, {}
for ln in sys.stdin:
    m = re.match(r"(\S+):(\d+)\s+([\d.]+)/step\s+[\d.]+%\s+stalls\s+([\d.]+)%", ln)
    if not m:
        continue
    f, line, v, s = m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4))
    if fsub in f:
        k = "?"
        for start, name in marks:
            if line >= start:
                k = name
    else:
        k = f
    tot[k] = tot.get(k, 0) + v
    st[k] = st.get(k, 0) + s
for k in sorted(tot, key=lambda x: -tot[x]):
    print(f"{k:28s} {tot[k]:8.1f}  stalls {st[k]:5.1f}%")
print(f"{'TOTAL':28s} {sum(tot.values()):8.1f}")
