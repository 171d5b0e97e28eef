"""GAES v1 container wire format and record handling (no GPU).

Fixtures come from the reference itself (tests/golden/make_golden.py):
container_bytes of the test_container.py golden recipe (SHA-256 pinned at
test_container.py:26) and a 300-record file through cli._split_records +
pad_zero + encrypt_batch + container_bytes.
"""

import hashlib

import numpy as np
import pytest

from paper_1506_08503_b200 import container as C

GOLDEN_SHA256 = "9e8a98b50f59f03773b6990cb07a40b6a2f4e7c0b704e695c6987d3366ea673b"


def test_golden_container_digest_and_parse(golden):
    blob = golden["container_golden"].tobytes()
    assert hashlib.sha256(blob).hexdigest() == GOLDEN_SHA256
    ivm, ivs, lens, payload = C.unpack(blob)
    assert ivm == C.IV_SHARED and ivs.tobytes() == bytes.fromhex("f0e1d2c3b4a5968778695a4b3c2d1e0f")
    assert list(lens) == [5, 11, 24] and payload.shape == (3, 32)
    assert C.pack(ivm, ivs, lens, payload) == blob


def test_records_split_pad_matches_reference(golden):
    content = golden["records_content"].tobytes()
    grid, lens = C.split_records(content)
    blob = golden["records_shared_container"].tobytes()
    _, _, ref_lens, ref_payload = C.unpack(blob)
    assert np.array_equal(lens, ref_lens)
    assert grid.shape == ref_payload.shape
    # zero padding beyond each length, record bytes in place
    recs = content.split(b"\n")[:-1]
    for i in (0, 1, 150, 299):
        assert grid[i, :lens[i]].tobytes() == recs[i] and not grid[i, lens[i]:].any()
    assert C.join_records(grid, lens) == content
    assert C.join_records(grid, lens, raw=True) == b"".join(recs)


def test_per_message_container_round_trip(golden):
    blob = golden["records_permsg_container"].tobytes()
    ivm, ivs, lens, payload = C.unpack(blob)
    assert ivm == C.IV_PER_MESSAGE and np.array_equal(ivs, golden["records_ivs"])
    assert C.pack(ivm, ivs, lens, payload) == blob


@pytest.mark.parametrize("content,err", [(b"", "empty input"), (b"\n", "record 1 has zero length"),
                                         (b"a\n\nb", "record 2 has zero length")])
def test_record_errors(content, err):
    with pytest.raises(C.DataError, match=err):
        C.split_records(content)


def test_record_edge_cases():
    g, lens = C.split_records(b"abc")
    assert list(lens) == [3] and g.shape == (1, 16)
    g, lens = C.split_records(b"x" * 16 + b"\n" + b"y")
    assert list(lens) == [16, 1] and g.shape == (2, 16)
    g, lens = C.split_records(b"a\nb\n\n", raw=True)
    assert list(lens) == [5] and g[0, :5].tobytes() == b"a\nb\n\n"


def test_parse_errors_match_reference_messages(golden):
    blob = golden["container_golden"].tobytes()
    with pytest.raises(C.ContainerError, match="truncated header"):
        C.unpack(blob[:10])
    with pytest.raises(C.ContainerError, match="bad magic"):
        C.unpack(b"XAES" + blob[4:])
    with pytest.raises(C.ContainerError, match="unsupported version"):
        C.unpack(blob[:4] + b"\x02" + blob[5:])
    with pytest.raises(C.ContainerError, match="unknown IV mode"):
        C.unpack(blob[:6] + b"\x07" + blob[7:])
    with pytest.raises(C.ContainerError, match="nonzero reserved"):
        C.unpack(blob[:7] + b"\x01" + blob[8:])
    with pytest.raises(C.ContainerError, match="size mismatch"):
        C.unpack(blob + b"\x00")
    bad = bytearray(blob)
    bad[16 + 16:16 + 20] = (99).to_bytes(4, "big")  # first length > width
    with pytest.raises(C.ContainerError, match="length field out of range"):
        C.unpack(bytes(bad))
