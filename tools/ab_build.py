"""Build libnpm.so from another git revision for A/B timing on the GPU box.

usage: python tools/ab_build.py <rev> <out.so>
The output is loaded by the binding when NPM_LIB=<out.so> is set, so two
builds can be timed in the same gpurun call (run-to-run noise across boxes is
~1-2 %)."""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rev, out):
    tmp = tempfile.mkdtemp(prefix="npm_ab_")
    arch = subprocess.run(["git", "-C", ROOT, "archive", rev, "paper_2504_04315_b200/csrc", "include"],
                          capture_output=True, check=True).stdout
    subprocess.run(["tar", "-x", "-C", tmp], input=arch, check=True)
    csrc = os.path.join(tmp, "paper_2504_04315_b200", "csrc")
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo", "-Xcompiler",
             "-fPIC", "--expt-relaxed-constexpr", "-I" + os.path.join(tmp, "include"), "-I" + csrc]
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    objs = [s[:-3] + ".o" for s in srcs]
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda so: subprocess.run(["nvcc"] + flags + ["-c", so[0], "-o", so[1]], check=True),
                    zip(srcs, objs)))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out] + objs + ["-lcudart", "-ldl"],
                   check=True)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1], os.path.abspath(sys.argv[2]))
