"""Print the SASS of one kernel from a library: python tools/sass_fn.py LIB.so SUBSTRING [--all]
(the first function whose mangled name contains SUBSTRING; instructions only)."""
import re, subprocess, sys
lib, sub = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if sub in name:
        print("//", name)
        for ln in f.split("\n")[1:]:
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if m:
                print(m.group(1), m.group(2).strip())
        break
