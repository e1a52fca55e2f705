"""Build the Cython binding of INTEGRATION.md §3 (integration/_accel_b200*.so),
linked against paper_2203_08263_b200/libnbody_b200.so with an rpath."""
import os, subprocess, sys, sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
PKG = os.path.join(REPO, "paper_2203_08263_b200")


def build() -> str:
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    c_file = os.path.join(HERE, "_accel_b200.c")
    so = os.path.join(HERE, "_accel_b200" + ext)
    subprocess.run(["cython", "-3", "-o", c_file, os.path.join(HERE, "_accel_b200.pyx")], check=True)
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"],
                    "-I", os.path.join(REPO, "include"), "-o", so, c_file,
                    "-L", PKG, "-l:libnbody_b200.so", "-Wl,-rpath,$ORIGIN/../paper_2203_08263_b200"], check=True)
    return so


if __name__ == "__main__":
    print(build())
