"""CPU tests of the GNSG header/size checks (graph.py:302-343 error contract)."""

import numpy as np
import pytest

from paper_2106_06150_b200 import formats
from paper_2106_06150_b200._lib import GraphFormatError


def _write(path, n=3, e=4, fdim=0, body_delta=0, magic=b"GNSG", version=1):
    hdr = formats._HEADER.pack(magic, version, n, e, fdim, 0, 0)
    body = 8 * (n + 1) + 8 * e + 4 * n * fdim + body_delta
    path.write_bytes(hdr + b"\0" * max(body, 0))


def test_header_ok(tmp_path):
    p = tmp_path / "g.gnsg"
    _write(p)
    h = formats.read_header(p)
    assert h["num_nodes"] == 3 and h["num_edges"] == 4 and h["feature_dim"] == 0


@pytest.mark.parametrize("kw,msg", [(dict(magic=b"XXXX"), "bad magic"), (dict(version=2), "unsupported version"),
                                    (dict(body_delta=-8), "expected 64 bytes after header, got 56")])
def test_header_errors(tmp_path, kw, msg):
    p = tmp_path / "g.gnsg"
    _write(p, **kw)
    with pytest.raises(GraphFormatError, match=msg):
        formats.read_header(p)


def test_truncated_header(tmp_path):
    p = tmp_path / "g.gnsg"
    p.write_bytes(b"GNS")
    with pytest.raises(GraphFormatError, match="truncated header"):
        formats.read_header(p)


def test_reference_written_file_parses(tmp_path, gb):
    g = gb.generate_sbm(60, 3, 0.3, 0.05, seed=0, feature_dim=5)
    p = tmp_path / "ref.gnsg"
    gb.save_binary(g, p)
    h = formats.read_header(p)
    assert h == dict(num_nodes=60, num_edges=g.num_edges, feature_dim=5, has_labels=True, has_masks=True)
