"""A/B of programmatic dependent launch (LSB_TUNE_PDL) on the C3 sweep's
small sizes and the C2 cycle: python tools/pdl_ab.py [0|1] [c3 args...]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from paper_1809_05805_b200 import _abi  # noqa: E402

_abi.load().lsb_set_tuning(_abi.TUNE_PDL, int(sys.argv[1]))
sys.argv = [sys.argv[0]] + sys.argv[2:]
import c3_sweep  # noqa: E402

c3_sweep.main()
