"""CRC-32/IEEE computed one bit at a time (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:768-769 (§6.1 "Deadlock and Liveness"): "To detect data corruption, a
checksum is applied to the data header. The consumer verifies this checksum
upon reading; if a mismatch is detected, the data is discarded."  The paper
names no algorithm; reading R10 takes the standard CRC-32 (the
zlib / IEEE 802.3 one: reflected polynomial 0xEDB88320, init 0xFFFFFFFF,
final xor 0xFFFFFFFF), as SPEC.md:249 ("standard CRC-32") does.

Pins (tests/test_oracle_crc.py): check value crc32(b"123456789") = 0xCBF43926
(the published check value of CRC-32/ISO-HDLC), crc32(b"") = 0, agreement with
the independent library routine zlib.crc32, and every single-bit flip of a
64-byte sample changes the result.
"""

POLY_REFLECTED = 0xEDB88320


def crc32(data: bytes) -> int:
    """Textbook shift-register CRC-32, LSB-first, one bit per iteration."""
    reg = 0xFFFFFFFF
    for byte in bytes(data):
        reg ^= byte
        for _ in range(8):
            if reg & 1:
                reg = (reg >> 1) ^ POLY_REFLECTED
            else:
                reg >>= 1
    return reg ^ 0xFFFFFFFF
