"""Run the reference's own hot-path tests unchanged against the B200 package.

`dbf`, `dbf.bitcore` and `dbf.kernel` are aliased to paper_2505_11076_b200 (the drop-in surface the
reference tests import), and the helpers below restate /root/reference/pkg/tests/conftest.py:7-25
(`random_signs`, `random_layer`, the `rng` fixture).  Every test here computes on the GPU (pack,
sign_matvec and forward run the sm_100a kernels), so the directory is marked `gpu`.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[2]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2505_11076_b200 as _pkg  # noqa: E402
from paper_2505_11076_b200 import bitcore as _bitcore, kernel as _kernel  # noqa: E402

sys.modules.setdefault("dbf", _pkg)
sys.modules.setdefault("dbf.bitcore", _bitcore)
sys.modules.setdefault("dbf.kernel", _kernel)



def pytest_collection_modifyitems(config, items):
    here = Path(__file__).resolve().parent
    for item in items:
        if Path(str(item.fspath)).resolve().parent == here:
            item.add_marker(pytest.mark.gpu)


# The reference tests import helpers with `from conftest import ...`, and pytest keeps ONE module
# named `conftest` for both directories: re-export every helper of tests/conftest.py from here
# (random_signs, f32_vector, random_layer restate pkg/tests/conftest.py:7-24), so whichever
# conftest is current serves both suites.
import importlib.util  # noqa: E402

_spec = importlib.util.spec_from_file_location("_dbf_tests_conftest", ROOT / "tests" / "conftest.py")
_root = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_root)
globals().update({k: v for k, v in vars(_root).items()
                  if not k.startswith("_") and not k.startswith("pytest_") and k not in globals()})
