"""Group compute-sanitizer racecheck (analysis mode) reports by kernel and the pair of source
locations, so every reported race is accounted for (the first 100 were not enough)."""
import re
import sys
from collections import Counter

txt = open(sys.argv[1], errors="replace").read()
blocks = re.split(r"\n========= (?=(?:Error|Warning): Race reported)", txt)
cnt = Counter()
for b in blocks:
    if "Race reported" not in b:
        continue
    locs = re.findall(r"at ([\w:<>,\s\*\(\)&]+?)\+0x[0-9a-f]+ in ([\w./]+:\d+)", b)
    kern = ""
    m = re.search(r"in (?:void )?(ws::[\w<>, ]+)", b)
    if m:
        kern = m.group(1)
    key = (kern, tuple(sorted(set(l[1].split("/")[-1] for l in locs))))
    cnt[key] += 1
for (kern, locs), n in cnt.most_common():
    print("%7d  %-40s %s" % (n, kern[:40], " <-> ".join(locs)))
print("total reports", sum(cnt.values()))
