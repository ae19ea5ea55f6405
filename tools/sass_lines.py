"""Static SASS instruction count per source line of one kernel in a cubin
(development tool: code-size / i-cache budget).
Usage: python tools/sass_lines.py CUBIN KERNEL_SUBSTRING [top]"""
import collections
import re
import subprocess
import sys

cubin, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True,
                     text=True).stdout
cnt = collections.Counter()
cur = None
on = False
for line in txt.splitlines():
    if line.strip().startswith(".text.") and line.rstrip().endswith(":"):
        on = pat in line
    if line.lstrip().startswith("//## File"):
        f = re.search(r'File "([^"]+)"', line)
        m = re.search(r"line (\d+)", line)
        cur = (f.group(1).split("/")[-1] if f else "?", int(m.group(1)) if m else -1)
        continue
    if on and re.search(r"/\*[0-9a-f]{4}\*/", line):
        cnt[cur] += 1
print(sum(cnt.values()), "instructions")
for k, v in cnt.most_common(top):
    print(f"{v:5d} {k[0]}:{k[1]}")
