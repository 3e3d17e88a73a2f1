"""Build the CPU oracle shared library (test infrastructure; see vpetabc_oracle.h)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libvpetabc_oracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "vpetabc_oracle.c")
    hdr = os.path.join(HERE, "vpetabc_oracle.h")
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return LIB
    # -ffp-contract=off: no FMA contraction, every FP64 op rounds as written.
    cmd = ["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", "-Wall", "-Wextra", "-o", LIB, src, "-lm"]
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
