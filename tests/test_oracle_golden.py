"""Oracle drift guard: BASELINE config 1 digests recorded by tests/golden/make_golden.py."""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))
from make_golden import digests  # noqa: E402


def test_oracle_golden_config1():
    want = json.loads((HERE / "golden" / "config1_golden.json").read_text())
    got = digests()
    for k, v in got.items():
        assert want[k] == v, k
