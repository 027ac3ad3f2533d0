"""GPU: the slab-decomposed grid (config 5 kernels and layouts) against the
oracle, for 1 rank and for 2 / 4 ranks emulated on one device."""
import numpy as np
import pytest

from helpers import config2_params, normwise_rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,ranks", [(256, 1), (256, 2), (256, 4), (1024, 2)])
def test_slab_matches_oracle(port, n, ranks):
    from paper_2503_03326_b200.slab import SlabSurface, emulated_frame
    p = config2_params(seed=7)
    L = 4096.0 * n / 16384  # config 5 resolution per metre, scaled down
    slabs = [SlabSurface(n, ranks, r, L, p) for r in range(ranks)]
    got = emulated_frame(slabs, 10.0)
    want = port.generate_maps(n, [L], [], p, 10.0)[0]
    for f in range(8):
        assert normwise_rel(got[f], want[f]) < 1e-4, f


@pytest.mark.parametrize("n,ranks", [(4096, 1), (4096, 2), (8192, 4)])
def test_slab_fourstep_matches_maps(n, ranks):
    """n >= 4096: the four-step column pass (in place in the receive buffer)
    against the single-grid spectral path at the same size, which
    test_generate_maps_large pins to the oracle at 4096."""
    from paper_2503_03326_b200 import ocean as oc
    from paper_2503_03326_b200.slab import SlabSurface, emulated_frame
    p = config2_params(seed=7)
    L = 4096.0 * n / 16384
    slabs = [SlabSurface(n, ranks, r, L, p) for r in range(ranks)]
    got = emulated_frame(slabs, 10.0)
    cs = oc.CascadeSet(oc.CascadeConfig(n, [L], []), p)
    want = oc.generate_maps(cs, 10.0, oc.SurfaceGenOptions(choppiness=1.0)).all_fields()[0]
    for f in range(8):
        assert normwise_rel(got[f], want[f]) < 1e-4, f


@pytest.mark.parametrize("n", [1024, 8192])
def test_slab_frame_with_comm(port, n):
    """ocn_slab_frame through the library's NCCL communicator (one rank on this
    one-GPU box: the exchange is the rank's own tile copy) equals the separate
    row / column passes, and matches the oracle at 1024."""
    import torch
    from paper_2503_03326_b200.slab import Comm, SlabSurface, emulated_frame, frame, tile_layout
    p = config2_params(seed=7)
    L = 4096.0 * n / 16384
    slab = SlabSurface(n, 1, 0, L, p)
    comm = Comm(slab.ctx, 1, 0)
    _, total = tile_layout(slab.rows, 1)
    send = torch.empty(2 * total, dtype=torch.float32, device="cuda:0")
    recv = torch.empty_like(send)
    frame(slab, comm, 10.0, send.data_ptr(), recv.data_ptr())
    slab.ctx.synchronize()
    got = np.stack([slab.field(f) for f in range(8)])
    ref = emulated_frame([SlabSurface(n, 1, 0, L, p)], 10.0)
    for f in range(8):
        assert normwise_rel(got[f], ref[f]) < 1e-6, f
    if n == 1024:
        want = port.generate_maps(n, [L], [], p, 10.0)[0]
        for f in range(8):
            assert normwise_rel(got[f], want[f]) < 1e-4, f
