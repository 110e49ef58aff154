"""ctypes binding of oracle/_ref/libigabem_ref.so -- TEST INFRASTRUCTURE ONLY.

The reference itself (igabem core sources compiled unmodified against the
Eigen-subset shim, see oracle/ref.mk and oracle/ref_harness.cpp), exposed with
the same Python interface as pyoracle (the restatement).  Used to pin the
oracle, to generate tests/golden/, and as bench.py's `kind: "reference"` CPU
baseline.  Loaded as an independent module instance of pyoracle's code."""
import importlib.util
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_spec = importlib.util.spec_from_file_location("oracle._pyref_impl", os.path.join(_HERE, "pyoracle.py"))
_mod = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mod)
_mod.LIB_PATH = os.path.join(_HERE, "_ref", "libigabem_ref.so")
_mod.PREFIX = "ref_"

lib = _mod.lib
gauss = _mod.gauss
pair_rule = _mod.pair_rule
admissible = _mod.admissible
Discretization = _mod.Discretization
H2Matrix = _mod.H2Matrix
KIND = _mod.KIND
FAR, VERTEX, EDGE, COINCIDENT = _mod.FAR, _mod.VERTEX, _mod.EDGE, _mod.COINCIDENT


def available():
    return os.path.exists(_mod.LIB_PATH)
