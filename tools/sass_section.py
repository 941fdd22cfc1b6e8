"""Print the SASS of one kernel from `cuobjdump -sass` output (stdin)."""
import re
import sys

want = sys.argv[1]
on = False
for line in sys.stdin:
    if "Function :" in line:
        on = want in line
    if on:
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
        if m:
            print(m.group(1), m.group(2).strip())
