"""Run a script with paper_2605_09755_b200 bound to an alternate libskp.so (A/B probes only)."""
import runpy, sys
sys.path.insert(0, ".")
import paper_2605_09755_b200._lib as L
L.LIB_PATH = sys.argv[1]
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
