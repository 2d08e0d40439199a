"""Build libcodedinv.so of a git revision into ab/lib_<name>.so for same-box A/B timing
(python scripts/ab_build.py HEAD base; the working tree builds with name 'work')."""
import os, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2106_06445_b200"))
import build as B  # noqa: E402

rev, name, extra = sys.argv[1], sys.argv[2], sys.argv[3:]   # extra: nvcc flags, e.g. -DFOO
out = os.path.join(ROOT, "ab", f"lib_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
with tempfile.TemporaryDirectory() as d:
    if rev == "work":
        src_root = ROOT
    else:
        subprocess.check_call(f"git -C {ROOT} archive {rev} paper_2106_06445_b200/csrc include | tar -x -C {d}", shell=True)
        src_root = d
    csrc = os.path.join(src_root, "paper_2106_06445_b200", "csrc")
    objs = []
    for f in sorted(os.listdir(csrc)):
        if f.endswith(".cu"):
            o = os.path.join(d, f + ".o")
            subprocess.check_call([B.NVCC, *B.FLAGS, *extra, "-I", os.path.join(src_root, "include"), "-I", csrc, "-c",
                                   os.path.join(csrc, f), "-o", o], stderr=subprocess.DEVNULL)
            objs.append(o)
    subprocess.check_call([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, "-lcuda"])
print(out)
