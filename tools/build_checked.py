"""Build paper_1210_5093_b200/libdfa_checked.so: the library with -DDFA_CHECKED (device-side
bounds checks on every table lookup, data-dependent index and input read; a violation prints
its site and traps).  Used by tools/checked_run.sh in place of compute-sanitizer, which the
B200 pool refuses."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("dfa_build", os.path.join(ROOT, "paper_1210_5093_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
print(b.build(force="--force" in sys.argv, lib=os.path.join(b.HERE, "libdfa_checked.so"), defines=("DFA_CHECKED",)))
