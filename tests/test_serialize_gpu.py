"""H2M1 container of device matrices (serialize.hpp), restated from the
reference's test_serialize.cpp, plus an independent parse of the byte layout
the reference defines (magic, version, tagged sections) to pin compatibility."""
import struct

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import (Admissibility, H2Matrix, build_block_tree, build_cluster_tree, deserialize,
                                   io_error, read_h2_file, serialize, write_h2_file)

pytestmark = pytest.mark.gpu


def make(sym, weak=False):
    pts = O.grid2d(24, 24) if not weak else O.grid1d(300, -1, 1)
    leaf = 16
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    ref = O.Tree(pts, leaf, 1.0, weak)
    ora = O.H2.random(ref, sym, 7, 31)
    rr, cr = ora.ranks()
    return H2Matrix.from_packed(bt, sym, rr, cr, ora.export()), ora, pts


@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("weak", [False, True])
def test_round_trip_bit_exact(cuda, sym, weak):   # test_serialize.cpp:23-47
    m, _, pts = make(sym, weak)
    b1 = serialize(m)
    m2 = deserialize(b1)
    assert serialize(m2) == b1
    p1, p2 = m.download(), m2.download()
    assert all(np.array_equal(p1[k], p2[k]) for k in p1)
    assert np.array_equal(m.ranks()[0], m2.ranks()[0])
    assert m2.symmetric == sym
    # bitwise matvec after the round trip (test_serialize.cpp:49-60)
    x = O.gaussian(3, pts.shape[0], 5)
    assert np.array_equal(m.matvec(x), m2.matvec(x))
    assert np.array_equal(m2.blocks.tree.perm, m.blocks.tree.perm)


def test_file_round_trip(cuda, tmp_path):
    m, _, pts = make(True)
    f = tmp_path / "m.h2m1"
    write_h2_file(m, f)
    m2 = read_h2_file(f)
    x = O.gaussian(4, pts.shape[0], 3)
    assert np.array_equal(m.matvec(x), m2.matvec(x))


def test_error_kinds(cuda):   # test_serialize.cpp:62-100
    m, _, _ = make(True)
    b = serialize(m)
    with pytest.raises(io_error) as e:
        deserialize(b"XXXX" + b[4:])
    assert e.value.kind == "bad_magic"
    with pytest.raises(io_error) as e:
        deserialize(b[:4] + struct.pack("<I", 2) + b[8:])
    assert e.value.kind == "version_mismatch"
    with pytest.raises(io_error) as e:
        deserialize(b[:len(b) // 2])
    assert e.value.kind == "truncated"
    with pytest.raises(io_error) as e:
        deserialize(b + struct.pack("<IQ", 99, 0))
    assert e.value.kind == "malformed"


def parse_h2m1(b):
    """Independent reader of the reference layout (serialize.hpp:26-182)."""
    assert b[:4] == b"H2M1"
    (ver,) = struct.unpack_from("<I", b, 4)
    at, secs = 8, {}
    while at < len(b):
        tag, ln = struct.unpack_from("<IQ", b, at)
        at += 12
        secs[tag] = b[at:at + ln]
        at += ln
    return ver, secs


def test_layout_matches_reference_spec(cuda):
    m, ora, pts = make(True)
    ver, secs = parse_h2m1(serialize(m))
    assert ver == 1 and set(secs) == {1, 2, 3, 4, 6, 7}   # no column basis for symmetric matrices
    ct = secs[1]
    n, dim, leaf, nv = struct.unpack_from("<qiqi", ct, 0)
    assert (n, dim, leaf) == (pts.shape[0], 2, 16) and nv == m.blocks.tree.num_nodes
    rec = 8 + 8 + 4 * 4 + 2 * 8 * dim
    perm = np.frombuffer(ct, "<i8", count=n, offset=24 + nv * rec)
    assert np.array_equal(perm, O.Tree(pts, 16, 1.0, False).perm)
    eta, weak, nodes, nadm, ndense = struct.unpack_from("<dBqqq", secs[2], 0)
    assert eta == 1.0 and weak == 0 and nadm == len(m.blocks.admissible_leaves)
    assert struct.unpack_from("<BB", secs[3], 0) == (1, 0)
    # couplings: (int32 block id, int64 rows, int64 cols, doubles) for canonical blocks in admissible order
    s = secs[6]
    (count,) = struct.unpack_from("<q", s, 0)
    bt = m.blocks
    canon = [b for b in bt.admissible_leaves if bt.row[b] <= bt.col[b]]
    assert count == len(canon)
    at = 8
    S = ora.export()["S"]
    so = 0
    rr, _ = ora.ranks()
    for b in canon[:50]:
        blk, r, c = struct.unpack_from("<iqq", s, at)
        at += 20
        assert blk == b and (r, c) == (rr[bt.row[b]], rr[bt.col[b]])
        vals = np.frombuffer(s, "<f8", count=r * c, offset=at)
        assert np.array_equal(vals, S[so:so + r * c])
        at += 8 * r * c
        so += r * c
