"""Attribute the SASS of one kernel to source lines (code-size debugging).

  python tools/sass_lines.py build/score_fused.o k_fusedILi4E [N]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    cnt = collections.Counter()
    infn, cur, src_file = False, None, None
    for line in txt.split("\n"):
        if line.startswith(".text."):
            infn = pat in line
        m = re.search(r'//## File "([^"]+)", line (\d+)( inlined at "[^"]+", line (\d+))?', line)
        if m:
            src_file = m.group(1)
            cur = int(m.group(4)) if m.group(4) else int(m.group(2))
            continue
        if infn and cur is not None and re.search(r"/\*[0-9a-f]{4,5}\*/", line):
            cnt[cur] += 1
    src = open(src_file).read().split("\n") if src_file else []
    print("total", sum(cnt.values()))
    for k, v in cnt.most_common(top):
        print(f"{v:6d} {k:5d} {src[k - 1].strip()[:100] if k <= len(src) else ''}")


if __name__ == "__main__":
    main()
