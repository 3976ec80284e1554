"""Static check: no module reads a name it never binds (catches NameErrors
on code paths that only run on the GPU box)."""
import subprocess
import sys

from conftest import ROOT


def test_no_undefined_names():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "lint_names.py"),
                        str(ROOT / "paper_2601_19489_b200"), str(ROOT / "bench.py"),
                        str(ROOT / "__graft_entry__.py"), str(ROOT / "tests"), str(ROOT / "oracle")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
