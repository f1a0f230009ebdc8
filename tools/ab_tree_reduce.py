"""tools/reduce_phases.py's 64 MiB block_reduce_f32 breakdown for the
package under argv[1] (two-tree A/B, see tools/ab_tree.py)."""
import os
import runpy
import sys

root = os.path.abspath(sys.argv[1])
sys.path.insert(0, root)
import paper_2310_01212_b200  # noqa: E402,F401
assert paper_2310_01212_b200.__file__.startswith(root)
sys.argv = ["reduce_phases.py"] + sys.argv[2:]
print(root, flush=True)
runpy.run_path(os.path.join(os.path.dirname(__file__), "reduce_phases.py"), run_name="__main__")
