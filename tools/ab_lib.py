"""A/B: run one_step with an alternative engine library (path in argv[1])."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_04424_b200 import _native
_native.LIB_PATH = os.path.abspath(sys.argv[1])
_native.load.__defaults__ = (_native.LIB_PATH,)
sys.argv = [sys.argv[0]] + sys.argv[2:]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "one_step.py")).read())
