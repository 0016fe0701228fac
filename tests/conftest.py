"""Shared test configuration.

Markers: ``gpu`` = needs a B200 and the built CUDA library (run with -m gpu);
everything else runs on CPU (oracle vs golden fixtures, host logic, C-ABI
export checks, gloo multi-process tests).
"""

import os
import sys


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)



def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (B200) and the built libpaball_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")
