"""Build the oracle's C scan (test infrastructure only) into oracle/_build/."""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build(force: bool = False) -> str:
    out_dir = os.path.join(HERE, "_build")
    os.makedirs(out_dir, exist_ok=True)
    src = os.path.join(HERE, "scan_oracle.c")
    out = os.path.join(out_dir, "liboracle_scan.so")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    # x86-64-v3 (AVX2) runs on this container and on the GPU box's host.
    cmd = ["gcc", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fopenmp", "-shared",
           "-fPIC", src, "-o", out, "-lm"]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    print(build(force=True))
