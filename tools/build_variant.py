"""Build an experimental variant of libapo.so with source substitutions
(for A/B kernel timing only; never used by tests or bench).

    python tools/build_variant.py NAME 'file::old::new' ...
Output: tools/variants/libapo_NAME.so
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    name = sys.argv[1]
    src = os.path.join(ROOT, "paper_2406_18111_b200", "csrc")
    base = f"/tmp/apo_variant_{name}"
    shutil.rmtree(base, ignore_errors=True)
    tmp = os.path.join(base, "pkg", "csrc")
    shutil.copytree(src, tmp)
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(base, "include"))
    for spec in sys.argv[2:]:
        f, old, new = spec.split("@@") if "@@" in spec else spec.split("::")
        p = os.path.join(tmp, f)
        s = open(p).read()
        assert old in s, (f, old)
        open(p, "w").write(s.replace(old, new))
    out = os.path.join(ROOT, "tools", "variants")
    os.makedirs(out, exist_ok=True)
    sys.path.insert(0, ROOT)
    from paper_2406_18111_b200 import build as b
    objs = []
    for s in b.SOURCES:
        o = os.path.join(tmp, s.replace(".cu", ".o"))
        subprocess.check_call([b.NVCC, *b.FLAGS, "-c", os.path.join(tmp, s), "-o", o])
        objs.append(o)
    subprocess.check_call([b.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                           os.path.join(out, f"libapo_{name}.so"), *objs])


if __name__ == "__main__":
    main()
