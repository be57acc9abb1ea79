"""The input generator's torch form (device-side generation of the large bench
inputs) reproduces the numpy generator element for element."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("dist", ["signed", "unit", "int"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_matrix_torch_matches_numpy(dist, dtype):
    import torch
    ref = synth.matrix(synth.BASE_SEED + 5, 300, 517, dist=dist, dtype=dtype, r0=37, r1=301 - 1)
    got = synth.matrix_torch(synth.BASE_SEED + 5, 300, 517, dist=dist, dtype=dtype, r0=37, r1=300, device="cpu",
                             chunk_rows=100)
    assert np.array_equal(got.float().numpy(), ref)
    big = synth.matrix_torch(7, 1 << 20, 4096, r0=(1 << 20) - 3, device="cpu")     # 64-bit counters
    assert np.array_equal(big.numpy(), synth.matrix(7, 1 << 20, 4096, r0=(1 << 20) - 3))
