"""GPU parity of dts_sr_prepare (depth-SR front end) against the fp64
oracle O9: target within 1e-5 x range(low) (fp32 bicubic; R24), confidence within
1e-6 (fp32 exp of a closed form), and the SR pipeline (front end -> DTS solve) end to end."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import make_inputs, target_range  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("h,w,f", [(1, 1, 1), (1, 1, 4), (7, 9, 1), (7, 9, 2), (5, 3, 3), (64, 86, 16), (33, 17, 8)])
def test_sr_prepare_parity(h, w, f):
    rng = np.random.default_rng(h * 100 + w * 10 + f)
    low = rng.uniform(0.5, 10.0, (h, w)).astype(np.float32)
    tr, cr = oracle.sr_prepare(low, f)
    t, c = dts.dts_sr_prepare(torch.from_numpy(low).cuda(), f)
    torch.cuda.synchronize()
    t, c = t.cpu().numpy().astype(np.float64), c.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(t - tr)) <= 1e-5 * max(target_range(low), 1.0)
    assert np.max(np.abs(c - cr)) <= 1e-6
    th, ch = dts.dts_sr_prepare(low, f)  # host pointers: same kernels, staged
    assert np.array_equal(th.astype(np.float64), t) and np.array_equal(ch.astype(np.float64), c)


def test_sr_pipeline_c2_shape():
    """C2's 86 x 64 depth samples (taken at the 16 x 16 block centres of the C2 target) through
    the front end, then the DTS solve on the 1376 x 1024 guide: GPU vs oracle end to end."""
    g, t_full, _ = make_inputs("C2")
    low = np.ascontiguousarray(t_full[8::16, 8::16]).astype(np.float32)
    assert low.shape == (64, 86)
    tr, cr = oracle.sr_prepare(low, 16)
    ref = oracle.solve(g, tr.astype(np.float32), cr.astype(np.float32), 32.0, 0.08, 3, 0.99, 10)
    gd = torch.from_numpy(g).cuda()
    t, c = dts.dts_sr_prepare(torch.from_numpy(low).cuda(), 16)
    with dts.Solver(gd, 32.0, 0.08, 3) as s:
        out = s.solve(t, c, 0.99, 10)
    torch.cuda.synchronize()
    assert np.max(np.abs(out.cpu().numpy() - ref)) <= 1e-4 * target_range(tr)


def test_sr_prepare_argument_errors():
    low = torch.rand(4, 5, device="cuda")
    out = torch.empty(8, 10, device="cuda")
    with pytest.raises(dts.DTSError) as ei:
        dts.dts_sr_prepare(low, 0, out, torch.empty_like(out))
    assert ei.value.status == 1
    with pytest.raises(dts.DTSError) as ei:
        dts.dts_sr_prepare(low, 2, out, out)  # outputs alias
    assert ei.value.status == 1
