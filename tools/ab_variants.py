"""Build libnpm.so variants of the WORKING TREE with extra -D flags (same-box
A/B timing: NPM_LIB=ab/<name>.so).  usage: python tools/ab_variants.py name=-DX,-DY name2= ..."""
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.environ.get("NPM_AB_SRC", ROOT)   # another source tree (e.g. a `git archive` of HEAD)


def build(name, defs):
    tmp = tempfile.mkdtemp(prefix="npm_abv_")
    shutil.copytree(os.path.join(SRC, "paper_2504_04315_b200", "csrc"), os.path.join(tmp, "p", "csrc"))
    shutil.copytree(os.path.join(SRC, "include"), os.path.join(tmp, "include"))
    csrc = os.path.join(tmp, "p", "csrc")
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
             "--expt-relaxed-constexpr", "-I" + os.path.join(tmp, "include"), "-I" + csrc] + defs
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    objs = [s[:-3] + ".o" for s in srcs]
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda so: subprocess.run(["nvcc"] + flags + ["-c", so[0], "-o", so[1]], check=True),
                    zip(srcs, objs)))
    os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
    out = os.path.join(ROOT, "ab", name + ".so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out] + objs +
                   ["-lcudart", "-ldl"], check=True)
    return out


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, _, d = spec.partition("=")
        print(build(name, [x for x in d.split(",") if x]))
