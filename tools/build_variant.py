"""Build an experiment variant of the library under another name with extra -D flags,
e.g. python tools/build_variant.py libdfa_w768.so DFA_WIN16_MAX_THREADS=768; select it with
DFA_LIB=paper_1210_5093_b200/<name> (the binding loads DFA_LIB when set)."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("dfa_build", os.path.join(ROOT, "paper_1210_5093_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
print(b.build(force=True, lib=os.path.join(b.HERE, sys.argv[1]), defines=tuple(sys.argv[2:])))
