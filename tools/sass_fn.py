"""Print the SASS of one kernel from a cuobjdump -sass listing: python tools/sass_fn.py <so> <substring>."""
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
cur, keep = None, []
for line in out.splitlines():
    if "Function :" in line:
        cur = line.split("Function :")[1].strip()
    if cur and sys.argv[2] in cur:
        keep.append(line)
print("\n".join(keep))
