"""Build an experiment variant of libhmx.so with extra nvcc flags into build/ab/<name>.so

    python tools/build_variant.py NAME -DFLAG=1 ...
"""
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_09384_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
b.OBJ = os.path.join(root, "build", "var_" + name, "obj")
b.LIB = os.path.join(root, "build", "var_" + name, "libhmx.so")
b.FLAGS = [f for f in b.FLAGS if f] + flags
b.build(force=True, verbose=False)
os.makedirs(os.path.join(root, "build", "ab"), exist_ok=True)
shutil.copy(b.LIB, os.path.join(root, "build", "ab", name + ".so"))
shutil.rmtree(os.path.join(root, "build", "var_" + name))
print("built build/ab/%s.so" % name)
