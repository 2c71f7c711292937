"""Compile the current tree's libfastged.so into ab/<name>.so (A/B timing: FASTGED_LIB=ab/<name>.so)."""
import os, shutil, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import build
name = sys.argv[1]
build.NVCC_FLAGS.extend(sys.argv[2:])
os.makedirs("ab", exist_ok=True)
lib = build.build(force=True)
shutil.copy(lib, f"ab/{name}.so")
print("ab/%s.so" % name)
