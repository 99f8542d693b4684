"""paper_2605_08793_b200 -- B200-native entropic-OT dual solver (drop-in for the
reference's `regot` solver entry points).  See DESIGN.md and INTEGRATION.md."""
from .regot import *  # noqa: F401,F403
from .regot import Solver, SparseSym, default_solver  # noqa: F401
