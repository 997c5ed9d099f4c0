"""Build the plain C++ oracle (TEST INFRASTRUCTURE ONLY): g++ -O2, no BLAS/LAPACK.

    python -m oracle.cpp.build   ->  oracle/cpp/libtn_oracle.so
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tn_oracle.cpp")
LIB = os.path.join(HERE, "libtn_oracle.so")


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", LIB, SRC], check=True)
    return LIB


if __name__ == "__main__":
    print(build())
