"""The device generator (product) is bit-identical to the reference's generate()
(generator.hpp:46-83), checked against the oracle restatement (itself pinned to the
reference in test_oracle_pin.py)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("w,h,d,g,seed", [
    (2048, 2048, 0.5, 1, 1), (2048, 2048, 0.35, 16, 1), (1920, 1080, 0.73, 7, 5),
    (37, 29, 0.5, 3, 99), (33, 21, 0.37, 2, 123456789), (16, 16, 1.0, 4, 7), (16, 16, 0.0, 1, 7),
    (1001, 3, 0.5, 2, 4)])
def test_generate_matches_reference(w, h, d, g, seed):
    import torch
    from paper_2006_09299_b200.runlab import generate_device
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    generate_device(out.data_ptr(), w, h, d, g, seed)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), O.generate(w, h, d, g, seed))


def test_generate_rings_matches_oracle():
    import torch
    from paper_2006_09299_b200.runlab import generate_rings_device
    for (w, h, seed, salt) in [(512, 512, 3, 0.02), (300, 200, 9, 0.0), (4096, 256, 3, 0.02)]:
        out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
        generate_rings_device(out.data_ptr(), w, h, 64, seed, salt)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), O.generate_rings(w, h, 64, seed, salt))


def test_cfg4_params_match_oracle():
    from paper_2006_09299_b200.runlab import cfg4_params
    for i in range(64):
        assert cfg4_params(i) == O.cfg4_params(i)
