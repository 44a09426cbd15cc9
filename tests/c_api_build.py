"""Builds examples/c_api_demo.c (plain C99 against include/mcs.h, linked to the in-tree
libmcs.so) for the C-ABI tests."""
import os
import subprocess

import paper_2504_18056_b200 as mcs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_demo(out_dir: str) -> str:
    lib = mcs.load()._name
    libdir = os.path.dirname(os.path.abspath(lib))
    exe = os.path.join(out_dir, "c_api_demo")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-pedantic",
           "-I" + os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "c_api_demo.c"),
           "-L" + libdir, "-l:" + os.path.basename(lib), "-Wl,-rpath," + libdir, "-lm", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe
