"""The per-iteration trace format (paper_1909_00145_b200/trace.py): CPU-only checks of the
row schema and the CSV round trip."""
import pytest

from paper_1909_00145_b200.trace import FIELDS, IterationTrace


def _row(i):
    return dict(iter=i, F=10.0 - i, fit=6.0 - i, l1=4.0, nnz=100 + i, tau_z=0.01, tau_d=0.5,
                ms_code=0.7, ms_filter=1.0, ms_obj=0.35, ms_iter=2.05)


def test_csv_round_trip():
    tr = IterationTrace()
    for i in range(5):
        tr.add(**_row(i))
    text = tr.to_csv()
    assert text.splitlines()[0] == ",".join(FIELDS)
    back = IterationTrace.read_csv(text)
    assert back.rows == tr.rows
    assert back.column("F") == [10.0, 9.0, 8.0, 7.0, 6.0]
    assert isinstance(back.rows[0]["nnz"], int)


def test_exact_float_repr():
    tr = IterationTrace()
    r = _row(0)
    r["F"] = 0.1 + 0.2  # not representable in a short decimal
    tr.add(**r)
    assert IterationTrace.read_csv(tr.to_csv()).rows[0]["F"] == r["F"]


def test_schema_errors():
    tr = IterationTrace()
    bad = _row(0)
    del bad["nnz"]
    with pytest.raises(ValueError):
        tr.add(**bad)
    with pytest.raises(ValueError):
        tr.add(**_row(0), extra=1)
    with pytest.raises(ValueError):
        IterationTrace.read_csv("iter,F\n1,2\n")
