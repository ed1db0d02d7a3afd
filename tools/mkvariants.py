"""Build libapo variants from (file, old, new) substitutions given as a
Python literal on stdin: {"name": [(file, old, new), ...], ...}
(diagnostics; outputs tools/variants/libapo_<name>.so)."""
import ast
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_18111_b200 import build as b  # noqa: E402

spec = ast.literal_eval(sys.stdin.read())
for name, subs in spec.items():
    base = f"/tmp/apo_variant_{name}"
    shutil.rmtree(base, ignore_errors=True)
    tmp = os.path.join(base, "pkg", "csrc")
    shutil.copytree(os.path.join(ROOT, "paper_2406_18111_b200", "csrc"), tmp)
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(base, "include"))
    for f, old, new in subs:
        p = os.path.join(tmp, f)
        s = open(p).read()
        assert old in s, (name, f, old[:60])
        open(p, "w").write(s.replace(old, new))
    objs = []
    for src in b.SOURCES:
        o = os.path.join(tmp, src.replace(".cu", ".o"))
        subprocess.check_call([b.NVCC, *b.FLAGS, "-c", os.path.join(tmp, src), "-o", o])
        objs.append(o)
    out = os.path.join(ROOT, "tools", "variants")
    os.makedirs(out, exist_ok=True)
    subprocess.check_call([b.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                           os.path.join(out, f"libapo_{name}.so"), *objs])
    print("built", name, flush=True)
