"""Group compute-sanitizer racecheck (analysis mode) reports by function and the pair of source
locations, summing the hazard counts, so every reported race is accounted for (the
first 100 hazards of the hazard mode were not enough)."""
import re
import sys
from collections import Counter

txt = open(sys.argv[1], errors="replace").read()
reports = re.split(r"\n========= (?=(?:Error|Warning): Race reported)", txt)
haz, rep = Counter(), Counter()
loc = re.compile(r"(Write|Read) access at (?:[\w ]+ )?(ws::.+?)\+0x[0-9a-f]+ in ([\w./]+:\d+)(?: \[(\d+) hazards?\])?")
for r in reports:
    if "Race reported" not in r:
        continue
    acc = loc.findall(r)
    if not acc:
        continue
    fn = re.sub(r"\(.*", "", acc[0][1])
    lines = tuple(sorted(set(a[2].split("/")[-1] for a in acc)))
    n = sum(int(a[3]) for a in acc if a[3]) or 1
    haz[(fn, lines)] += n
    rep[(fn, lines)] += 1
for k, n in haz.most_common():
    print("%9d hazards %5d reports  %-36s %s" % (n, rep[k], k[0][:36], " <-> ".join(k[1])))
print("total: %d hazards in %d reports" % (sum(haz.values()), sum(rep.values())))
