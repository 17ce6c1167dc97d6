import sys
sys.path.insert(0, ".")
from paper_1212_3032_b200 import _lib
_lib.load(sys.argv[1])
sys.argv = [sys.argv[0]]
exec(open("tools/gmres_overhead.py").read())
