"""Test helpers (importable as `fmm_testutil`; the name avoids clashing with other `tests` packages on sys.path)."""
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def golden(name: str) -> Path:
    return ROOT / "tests" / "golden" / name


def read_golden_matrices(name: str) -> dict:
    """Parse a tests/golden/*.txt file of named integer matrices (lines 'U', 'V', 'W' start a
    matrix; '#' lines are citations/comments)."""
    out, cur = {}, None
    for line in golden(name).read_text().splitlines():
        s = line.strip()
        if not s or s.startswith("#"):
            continue
        if s.isalpha():
            cur = s
            out[cur] = []
            continue
        out[cur].append([int(x) for x in s.split()])
    return out
