"""Timing-CSV compatibility: records written by
write_timing_csv (mirror of proj/src/engine.cpp:567-573) are read back by the
reference's own read_timing_csv (engine.cpp:575-601, via oracle/_ref)."""
import io

import pytest

import oracle as O


def _records(q):
    return [q.TimingRecord(0, 6, 12, 5, "b200", 1.25e-6, 32, 8 * 32 / 1.25e-6),
            q.TimingRecord(3, 7, 40, 26, "b200", 0.0003125, 1 << 26, 8.0 * (1 << 26) / 0.0003125)]


def test_roundtrip_python(q):
    buf = io.StringIO()
    q.write_timing_csv(_records(q), buf)
    text = buf.getvalue()
    assert text.splitlines()[0] == "edge_u,edge_v,bucket_seq,width,backend,elapsed_s,ops,flops_est"
    assert text.splitlines()[1] == "0,6,12,5,b200,1.25e-06,32,2.048e+08"
    back = q.read_timing_csv(io.StringIO(text))
    assert [(r.edge_u, r.edge_v, r.bucket_seq, r.width, r.backend, r.ops) for r in back] == \
           [(r.edge_u, r.edge_v, r.bucket_seq, r.width, r.backend, r.ops) for r in _records(q)]
    with pytest.raises(q.InvalidInputError, match="missing header"):
        q.read_timing_csv(io.StringIO(""))
    with pytest.raises(q.InvalidInputError, match="short row"):
        q.read_timing_csv(io.StringIO("h\n1,2,3\n"))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_reader_accepts_ours(q):
    buf = io.StringIO()
    recs = _records(q)
    q.write_timing_csv(recs, buf)
    n, wsum, ops = O.ref_read_timing_csv(buf.getvalue())
    assert (n, wsum, ops) == (len(recs), sum(r.width for r in recs), float(sum(r.ops for r in recs)))


@pytest.mark.gpu
def test_plan_records_csv(q, ctx, golden):
    c = golden["configs"]["C1"]
    g = q.random_regular(c["n"], 3, c["seed"])
    plan = q.Plan(g, 1, ctx=ctx)
    plan.execute(q.Angles(c["gammas"], c["betas"]))
    recs = plan.records()
    buf = io.StringIO()
    q.write_timing_csv(recs, buf)
    back = q.read_timing_csv(io.StringIO(buf.getvalue()))
    assert len(back) == c["n_records"] == len(recs)
    assert all(r.backend == "b200" and r.elapsed_s > 0 and r.ops == 1 << r.width for r in back)
    if O.ref_available():
        n, wsum, _ = O.ref_read_timing_csv(buf.getvalue())
        assert n == len(recs) and wsum == sum(r.width for r in recs)
