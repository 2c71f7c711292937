"""Compile the current tree's libfastged.so with extra nvcc flags into ab/<name>.so (A/B timing:
FASTGED_LIB=ab/<name>.so).  The in-tree product library is never touched."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import build
name = sys.argv[1]
os.makedirs("ab", exist_ok=True)
print(build.build(out=os.path.abspath(f"ab/{name}.so"), extra_flags=sys.argv[2:]))
