"""LOOKUP response frames: hps_wire_lookup_frame must be
byte-identical to the reference's encode_response_frame (wire.cpp:174-188)
with handle_frame's miss bitmap (server.cpp:284-294) -- the reference's own
KAT (test_wire.cpp:55-73), random frames vs the reference encoder, and the
device mode (bitmap packed on the GPU, rows copied straight from HBM into
the frame) vs the host mode."""
import numpy as np
import pytest

import oracle
import paper_2210_08804_b200 as hps


def test_reference_kat_lookup_response_frame():
    # test_wire.cpp:55-73
    want = bytes([0x12, 0, 0, 0, 0x00, 0x02, 0, 0, 0, 0x01, 0, 0, 0,
                  0x00, 0x00, 0x80, 0x3F, 0x00, 0x00, 0x20, 0xC0, 0x02])
    got = hps.wire_lookup_frame(np.array([1.0, -2.5], np.float32), np.array([0, 1], np.uint8), 1)
    assert got == want


@pytest.mark.parametrize("count,dim", [(0, 4), (1, 1), (7, 3), (8, 16), (9, 128), (1000, 5)])
def test_frames_match_reference_encoder(count, dim):
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(count * 31 + dim)
    rows = rng.standard_normal(count * dim).astype(np.float32)
    rows[::7] = -0.0
    flags = (rng.random(count) < 0.3).astype(np.uint8)
    assert hps.wire_lookup_frame(rows, flags, dim) == oracle.ref_wire_lookup_frame(rows, flags, dim)


@pytest.mark.gpu
@pytest.mark.parametrize("count,dim", [(1, 8), (31, 16), (33, 128), (65536, 128), (4099, 3)])
def test_device_frames_equal_host_frames(count, dim):
    import torch

    rng = np.random.default_rng(count + dim)
    rows = rng.standard_normal(count * dim).astype(np.float32)
    flags = (rng.random(count) < 0.2).astype(np.uint8)
    rt = torch.from_numpy(rows).cuda()
    ft = torch.from_numpy(flags).cuda()
    n = 13 + count * dim * 4 + (count + 7) // 8
    frame = torch.empty(n, dtype=torch.uint8).pin_memory()
    got_n = hps.wire_lookup_frame_device(rt.data_ptr(), ft.data_ptr(), count, dim,
                                         frame.data_ptr(), n)
    assert got_n == n
    assert frame.numpy().tobytes() == hps.wire_lookup_frame(rows, flags, dim)
