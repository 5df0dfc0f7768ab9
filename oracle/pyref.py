"""ORACLE — TEST INFRASTRUCTURE ONLY.

The reference's OWN code, compiled: oracle/_ref/libh2ref.so is oracle/capi.cpp
built with -DORA_REFERENCE_HEADERS against the unchanged headers under
/root/reference/proj/include/h2 (+ proj/tests/test_support.hpp) and the
Eigen-API shim in oracle/eigen_shim (`make -C oracle ref`, the reference's
Release flags from proj/CMakeLists.txt:3-20). This module exposes the same
Python API as oracle.pyoracle (Tree, H2, peel_dense, gaussian, ...) bound to
that library, so a test can run one check against the restatement and the
reference side by side.

Integer/index work (trees, permutations, block lists, RNG streams, sample
counts) is the reference's exactly. Floating-point results pass through the
shim's GEMM/QR/SVD, so they agree with an Eigen build to rounding, not bitwise.
"""
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB_PATH = os.path.join(_HERE, "_ref", "libh2ref.so")
_SRC = os.path.join(_HERE, "pyoracle.py")

_ns = {"__name__": __name__ + "._impl", "__file__": _SRC, "_LIB_OVERRIDE": REF_LIB_PATH}
with open(_SRC) as _f:
    exec(compile(_f.read(), _SRC, "exec"), _ns)

globals().update({k: v for k, v in _ns.items() if not k.startswith("__")})
