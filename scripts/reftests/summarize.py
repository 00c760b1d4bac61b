"""Per-file pass/fail counts from a pytest junit xml (reference-suite runs)."""

import collections
import json
import sys
import xml.etree.ElementTree as ET

root = ET.parse(sys.argv[1]).getroot()
per = collections.defaultdict(lambda: collections.Counter())
failed = []
for tc in root.iter("testcase"):
    f = tc.get("classname", "").split(".")[-1] or tc.get("file", "?")
    kind = "passed"
    for child in tc:
        if child.tag in ("failure", "error"):
            kind = "failed"
            failed.append(f"{f}::{tc.get('name')}: {(child.get('message') or '')[:160]}")
        elif child.tag == "skipped":
            kind = "skipped"
    per[f][kind] += 1
tot = collections.Counter()
for c in per.values():
    tot.update(c)
print(json.dumps({"total": dict(tot), "per_file": {k: dict(v) for k, v in sorted(per.items())},
                  "failed": failed}, indent=1))
