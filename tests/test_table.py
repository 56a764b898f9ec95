"""Autotuned configuration table (§5.2, SPEC tuner S:404-433): load,
exact and approximate lookup, tie-breaking, legality fallback in apt_select_config, and the
enumerated search space.  Host-only (no GPU)."""
import math

import pytest

P = pytest.importorskip("paper_2508_19087_b200")


def _row(m, n, k, wb, ab, cfg, us):
    keys = ("kernel", "w_digit", "a_digit", "bm", "bn", "bk", "stages", "split_k", "cta_pair", "cluster_n", "mma_kind")
    return " ".join(str(v) for v in (m, n, k, wb, ab, *(cfg[x] for x in keys), us))


@pytest.fixture
def empty_table():
    P.clear_table()
    yield
    P.clear_table()
    P.load_default_table()


def _write(tmp_path, rows, name="t.apt"):
    p = tmp_path / name
    p.write_text("# apt-table v1\n" + "\n".join(rows) + "\n")
    return str(p)


def _dec(m, wb, ab, warps=8, split=1):
    return dict(kernel=5, w_digit=wb, a_digit=ab, bm=32, bn=8 if m <= 8 else 16, bk=256, stages=warps, split_k=split,
                cta_pair=0, cluster_n=1, mma_kind=0)


def test_exact_hit_and_select(empty_table, tmp_path):
    cfg = _dec(16, 2, 2, 8, 1)
    assert P.load_table(_write(tmp_path, [_row(16, 4096, 4096, 2, 2, cfg, 5.0)])) == 1
    got, d = P.table_lookup(16, 4096, 4096, 2, 2)
    assert d == 0.0 and got == cfg
    assert P.select_config(16, 4096, 4096, 2, 2) == cfg


def test_approximate_matching_nearest_log2_key(empty_table, tmp_path):
    """a query absent from the table takes the nearest key by sum |log2| distance among rows with
    the same (wbits, abits)."""
    near, far = _dec(16, 2, 2, 8, 1), _dec(16, 2, 2, 4, 2)
    P.load_table(_write(tmp_path, [_row(16, 4096, 4096, 2, 2, near, 9.0), _row(16, 16384, 16384, 2, 2, far, 1.0),
                                   _row(16, 2048, 2048, 1, 1, _dec(16, 1, 1, 4, 3), 0.5)]))
    got, d = P.table_lookup(16, 2000, 2000, 2, 2)
    assert got == near
    assert math.isclose(d, 2 * abs(math.log2(2000) - math.log2(4096)), rel_tol=1e-12)
    # no row with (wbits, abits) = (3, 4): any row is a candidate
    got, d = P.table_lookup(16, 2048, 2048, 3, 4)
    assert got["split_k"] == 3 and d == 0.0


def test_tie_breaks_by_measured_time(empty_table, tmp_path):
    a, b = _dec(16, 2, 2, 8, 1), _dec(16, 2, 2, 4, 2)
    P.load_table(_write(tmp_path, [_row(16, 2048, 4096, 2, 2, a, 7.0), _row(16, 8192, 4096, 2, 2, b, 3.0)]))
    got, d = P.table_lookup(16, 4096, 4096, 2, 2)  # log2 distance 1 to both
    assert d == 1.0 and got == b


def test_later_rows_replace_and_bad_files(empty_table, tmp_path):
    a, b = _dec(16, 2, 2, 8, 1), _dec(16, 2, 2, 4, 2)
    P.load_table(_write(tmp_path, [_row(16, 4096, 4096, 2, 2, a, 7.0)], "a.apt"))
    assert P.load_table(_write(tmp_path, [_row(16, 4096, 4096, 2, 2, b, 6.0)], "b.apt")) == 1
    assert P.table_lookup(16, 4096, 4096, 2, 2)[0] == b
    with pytest.raises(RuntimeError, match="INVALID"):
        P.load_table(_write(tmp_path, ["16 4096 4096 2 2 5 2 2"], "bad.apt"))
    with pytest.raises(RuntimeError, match="INVALID"):
        P.load_table(str(tmp_path / "missing.apt"))
    assert P.table_size() == 1


def test_regimes_and_illegal_rows_fall_back_to_analytic(empty_table, tmp_path):
    """Rows of another token regime (decode M <= 16 vs prefill) never match; a matched row that is illegal
    for the queried shape (a DEC row for M = 9..16 asked at M = 12 with bn 8 -> illegal) falls back to the
    analytic rules."""
    analytic = P.select_config(2048, 4096, 4096, 4, 4)
    P.load_table(_write(tmp_path, [_row(16, 4096, 4096, 4, 4, _dec(16, 4, 4), 5.0)]))
    assert P.table_lookup(2048, 4096, 4096, 4, 4) is None
    assert P.select_config(2048, 4096, 4096, 4, 4) == analytic
    P.clear_table()
    analytic = P.select_config(12, 4096, 4096, 4, 4)
    P.load_table(_write(tmp_path, [_row(8, 4096, 4096, 4, 4, _dec(8, 4, 4), 5.0)]))
    assert P.table_lookup(12, 4096, 4096, 4, 4)[0]["bn"] == 8
    assert P.select_config(12, 4096, 4096, 4, 4) == analytic


def test_empty_table_lookup(empty_table):
    assert P.table_lookup(16, 4096, 4096, 2, 2) is None


@pytest.mark.parametrize("m,n,k,wb,ab", [(1, 4096, 4096, 1, 2), (8, 11008, 4096, 3, 4), (16, 4096, 11008, 4, 4),
                                         (2048, 4096, 4096, 2, 8), (4096, 8192, 8192, 2, 4), (37, 131, 700, 5, 3)])
def test_enumeration_is_the_legal_space(empty_table, m, n, k, wb, ab):
    """The search space holds only legal configs (each one selected through a one-row table is returned
    unchanged by apt_select_config, i.e. it passed the library's legality check), is free of duplicates,
    and contains the analytic choice."""
    space = P.enumerate_configs(m, n, k, wb, ab)
    assert space and len({tuple(sorted(c.items())) for c in space}) == len(space)
    assert P.select_config(m, n, k, wb, ab) in space
    for c in space[:: max(1, len(space) // 12)]:
        assert c["w_digit"] == wb and c["a_digit"] == ab
        if m <= 16:
            assert all(x["kernel"] in (2, 3, 4, 5, 6) for x in space)
    assert P.enumerate_configs(2, 33025, 33025, 8, 8) == []  # int32 bound (reading Q8)


def test_enumerated_configs_round_trip_through_table(empty_table, tmp_path):
    m, n, k, wb, ab = 8, 4096, 4096, 2, 2
    for c in P.enumerate_configs(m, n, k, wb, ab):
        P.clear_table()
        P.load_table(_write(tmp_path, [_row(m, n, k, wb, ab, c, 1.0)]))
        assert P.select_config(m, n, k, wb, ab) == c
