"""SASS of one kernel instantiation from an object file: python scripts/sass_fn.py obj regex [--dump]"""
import re, subprocess, sys
obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if re.search(pat, name):
        ins = [l for l in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l)]
        print(name[-60:], len(ins))
        if "--dump" in sys.argv:
            for l in ins: print(l.strip())
