"""Pins for the oracle's checksum and header encoding (CPU only).

The oracle's CRC is pinned to things other than itself: the published check
value of CRC-32/ISO-HDLC, the independent library routine zlib.crc32, and the
single-bit-flip property.  The header byte map is pinned by
assembling expected bytes with `struct` + zlib in the test (PAPER.md:419-425
fields in SPEC.md:261 order; R10/R11)."""
import random
import struct
import zlib

from oracle.crc32 import crc32
from oracle.ring import encode_header, decode_header, CRC_END


def test_crc_check_values():
    assert crc32(b"") == 0x00000000
    assert crc32(b"123456789") == 0xCBF43926


def test_crc_matches_zlib():
    rng = random.Random(1)
    for n in list(range(0, 70)) + [127, 128, 129, 1000]:
        b = bytes(rng.randrange(256) for _ in range(n))
        assert crc32(b) == zlib.crc32(b)


def test_crc_single_bit_flips_detected():
    rng = random.Random(2)
    sample = bytes(rng.randrange(256) for _ in range(64))
    base = crc32(sample)
    for i in range(64 * 8):
        m = bytearray(sample)
        m[i // 8] ^= 1 << (i % 8)
        assert crc32(bytes(m)) != base


def test_header_byte_map():
    uid = bytes(range(1, 17))
    h = encode_header(uid, 0x0102030405060708, 7, 3, 4194304, producer_id=1, seq=42, epoch=5, flags=0,
                      t_put=123456789)
    assert len(h) == 64
    # Independent assembly of the documented byte map.
    body = (uid + (0x0102030405060708).to_bytes(8, "little") + (7).to_bytes(4, "little")
            + (3).to_bytes(2, "little") + (4194304).to_bytes(4, "little") + bytes(6)
            + (1).to_bytes(4, "little") + (42).to_bytes(4, "little") + (5).to_bytes(2, "little")
            + (0).to_bytes(2, "little"))
    assert len(body) == 52
    expect = struct.pack("<I", zlib.crc32(body)) + body + (123456789).to_bytes(8, "little")
    assert h == expect
    d = decode_header(h)
    assert d["crc_ok"] and d["seq"] == 42 and d["producer_id"] == 1 and d["payload_len"] == 4194304
    assert d["epoch"] == 5 and d["t_put"] == 123456789 and d["uid"] == uid


def test_header_crc_coverage():
    h = bytearray(encode_header(bytes(16), 1, 2, 3, 4, 5, 6, 7, 8, t_put=99))
    for i in range(4 * 8, CRC_END * 8):
        m = bytearray(h)
        m[i // 8] ^= 1 << (i % 8)
        assert not decode_header(bytes(m))["crc_ok"]
    for i in range(CRC_END * 8, 64 * 8):    # t_put is outside the checksum (R10)
        m = bytearray(h)
        m[i // 8] ^= 1 << (i % 8)
        assert decode_header(bytes(m))["crc_ok"]
    for i in range(0, 32):                  # a corrupted stored CRC is detected
        m = bytearray(h)
        m[i // 8] ^= 1 << (i % 8)
        assert not decode_header(bytes(m))["crc_ok"]
