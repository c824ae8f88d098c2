"""Print the SASS of the kernels of a cubin/.o/.so whose demangled name contains a pattern.

Used to check that the unmelded forms keep their divergent branches and the melded
forms keep hoisted code + selects.
"""
import re
import subprocess
import sys


def sass_functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    dem = subprocess.run(["c++filt"], input=out, capture_output=True, text=True, check=True).stdout
    funcs = {}
    for chunk in re.split(r"\n\s*Function : ", dem)[1:]:
        lines = chunk.split("\n")
        body = []
        for line in lines[1:]:
            m = re.match(r"\s*/\*([0-9a-f]{4})\*/\s*(.*?);", line)
            if m and "NOP" not in m.group(2):
                body.append((m.group(1), re.sub(r"\s+", " ", m.group(2))))
        funcs[lines[0].strip()] = body
    return funcs


if __name__ == "__main__":
    path, pat = sys.argv[1], sys.argv[2]
    for name, body in sass_functions(path).items():
        if pat in name:
            print("=== " + name)
            for addr, ins in body:
                print(addr, ins)
