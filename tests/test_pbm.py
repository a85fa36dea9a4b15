"""PBM input/output (SURVEY 8(f) second row).  CPU part: the host-side header parser and the
P1 decoder against the reference's own read_pbm (error byte offsets, test_io.cpp:37-52), the P4
byte layout against write_pbm.  GPU part (-m gpu): P4 rasters decoded/encoded by the tile
kernels give exactly the byte-per-pixel results."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2006_09299_b200.runlab import PbmParseError, pack_p4, read_pbm_header

BAD = [b"P2\n3 1\n0 1 0\n", b"P1\nx 1\n", b"P1\n3 1\n0 1", b"P4\n9 2\n\x80\xff", b"P1\n0 4\n",
       b"P1\n99999999999 1\n", b"P1\n1048576 1048576\n", b"", b"P", b"Q4\n1 1\n\x00", b"P4\n2 2", b"P4\n2 2x\x00\x00",
       b"P4 # c\n8 # d\n1\n", b"P4\n8 1\n", b"P1\n2 1\n0 2\n", b"P1\n2 1\n# only comment"]
GOOD = [b"P1\n2 2\n0 1\n1 0\n", b"P1 # c\n3 # w\n1\n101", b"P4\n9 2\n\x80\xff\x00\xff",
        b"P4\t1 1 \x01", b"P4 # comment \n 16 1\n\xff\x00", b"P1\n1 1\n1"]

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("data", BAD)
def test_parse_errors_match_reference(data):
    _, off = O.ref_read_pbm(data)
    assert off is not None
    with pytest.raises(PbmParseError) as e:
        info = read_pbm_header(data)
        if info.format == 1:  # P1 raster errors surface while decoding
            _p1_pixels(data, info)
    assert e.value.byte_offset == off


def _p1_pixels(data, info):
    import ctypes as C
    from paper_2006_09299_b200 import _native as N
    rowb = (info.width + 7) // 8
    out = np.zeros(rowb * info.height, dtype=np.uint8)
    buf = C.create_string_buffer(bytes(data), len(data))
    rc = N.load().rl_pbm_p1_to_p4(buf, len(data), C.byref(info), out.ctypes.data_as(C.c_void_p))
    if rc == N.RL_EFORMAT:
        raise PbmParseError(info.message.decode(), int(info.error_offset))
    assert rc == 0
    return np.unpackbits(out.reshape(info.height, rowb), axis=1)[:, : info.width]


@needs_ref
@pytest.mark.parametrize("data", GOOD)
def test_parse_good_files_match_reference(data):
    px, off = O.ref_read_pbm(data)
    assert off is None
    info = read_pbm_header(data)
    assert (info.height, info.width) == px.shape
    if info.format == 1:
        np.testing.assert_array_equal(_p1_pixels(data, info), px)
    else:
        rowb = (info.width + 7) // 8
        rows = np.frombuffer(data, dtype=np.uint8, offset=info.raster_offset, count=rowb * info.height)
        np.testing.assert_array_equal(np.unpackbits(rows.reshape(info.height, rowb), axis=1)[:, : info.width], px)


@needs_ref
@pytest.mark.parametrize("w,h", [(1, 1), (7, 3), (9, 2), (37, 11), (256, 5), (1000, 3)])
def test_p4_layout_matches_write_pbm(w, h):
    import ctypes as C
    from paper_2006_09299_b200 import _native as N
    img = O.generate(w, h, 0.5, 1, w + h)
    ref = O.ref_write_pbm(img)
    hdr = C.create_string_buffer(64)
    n = N.load().rl_pbm_p4_header(w, h, hdr, 64)
    assert ref == hdr.raw[:n] + pack_p4(img).tobytes()
    px, _ = O.ref_read_pbm(O.ref_write_pbm(img, p1=True))
    np.testing.assert_array_equal(px, img)
