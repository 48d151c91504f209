"""Build an experimental variant of libsparse_mlp.so into build_ab/<tag>/ with extra nvcc flags
(e.g. -DSMLP_EXP_X=1), for A/B timing through SMLP_LIB=build_ab/<tag>/libsparse_mlp.so.  Not
part of the product: variants never ship in paper_2102_01732_b200/lib.

    python tools/ab_build.py <tag> [-Dflag ...]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2102_01732_b200 import build as B  # noqa: E402


def main():
    tag, flags = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "build_ab", tag)
    os.makedirs(out, exist_ok=True)

    def comp(src):
        obj = os.path.join(out, os.path.basename(src).replace(".cu", ".o"))
        subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *flags, "-c", src, "-o", obj], check=True, capture_output=True)
        return obj

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, B.sources()))
    lib = os.path.join(out, "libsparse_mlp.so")
    subprocess.run([B.nvcc(), "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                    "-o", lib], check=True)
    print(lib)


if __name__ == "__main__":
    main()
