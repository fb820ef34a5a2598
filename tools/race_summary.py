"""Fold a compute-sanitizer racecheck log (--print-limit 0) into counts per
(kernel, hazard kind, shared address, source line of each side)."""
import collections
import re
import sys

pat_h = re.compile(r"Error: Potential (\w+) hazard detected(?: \(([^)]*)\))? at __shared__ (0x[0-9a-f]+)")
pat_t = re.compile(r"(Write|Read) Thread \(([0-9,]+)\)(?: \(block rank (\d)\))? at void xnc::([A-Za-z_0-9]+)(<[^(]*)?.*?\+(0x[0-9a-f]+)(?: in ([\w.]+:\d+))?")
counts = collections.Counter()
cur = None
sides = []
n = 0
for line in open(sys.argv[1], errors="replace"):
    m = pat_h.search(line)
    if m:
        if cur:
            counts[cur + tuple(sides)] += 1
        cur = (m.group(1), m.group(2) or "", m.group(3))
        sides = []
        n += 1
        continue
    m = pat_t.search(line)
    if m and cur is not None:
        sides.append(f"{m.group(1)}:{m.group(4)}{m.group(5) or ''}@{m.group(7) or m.group(6)}"
                     f"{' rank' + m.group(3) if m.group(3) else ''}")
if cur:
    counts[cur + tuple(sides)] += 1
print(f"hazards parsed: {n}")
by_kernel = collections.Counter()
for k, c in counts.items():
    kern = k[3].split("@")[0].split(":", 1)[1] if len(k) > 3 else "?"
    by_kernel[kern] += c
print("per kernel:")
for k, c in by_kernel.most_common():
    print(f"  {c:8d}  {k}")
print("per (kind, note, shared address, write side, read side):")
for k, c in counts.most_common(60):
    print(f"  {c:8d}  {' | '.join(k)}")
for line in open(sys.argv[1], errors="replace"):
    if "SUMMARY" in line or ": ok" in line:
        print(line.rstrip())
