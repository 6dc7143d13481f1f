"""Parity at the BASELINE configs' FULL sizes — the configurations the bench
numbers are quoted on — against the CPU oracle fanned out over the host's
cores (tests/pool_oracle.py, identical results to the single-process
oracle, tests/test_pool_oracle.py):

  * C2 (configs[2]): 2^30 fp32, block 2^20, m = 16, Adam-m and Adam-v: all
    1024 cluster tables bit-equal; labels and codes of 64 spread blocks equal;
    their dequantized values bit-equal (quantizer.py:100-204);
  * per-tensor units of C3 / C4 size (configs[3-4], block = 0, the store's
    layout): a 32000 x 8192 = 262,144,000-element Adam-v tensor (C4's embed /
    lm_head) and a 4096 x 11008 Adam-m tensor (C3's MLP): table, labels and
    codes equal to the oracle's;
  * C1 (configs[1]): 2^30 bf16 at p = 0.1 / 1 / 6.25 / 25 %: the mask and the
    payload equal to the oracle's delta_encode (bitmask.py:94-111), and the
    decode restores the current tensor.
"""

import numpy as np
import pytest

from oracle import bitsnap_oracle as O
import pool_oracle as PO

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _tables_equal(host_table, ora, where=""):
    f = lambda v: np.asarray(v, np.float32).view(np.uint32).tolist()
    assert host_table.m == ora["m"], where
    assert f([host_table.mean, host_table.std]) == f([ora["mean"], ora["std"]]), where
    assert f(host_table.boundaries) == f(ora["boundaries"]), where
    assert f(host_table.scales) == f(ora["scales"]), where
    assert f(host_table.offsets) == f(ora["offsets"]), where


@pytest.mark.parametrize("dist", ["adam_m", "adam_v"])
def test_c2_all_blocks_vs_oracle(dev, dist):
    import torch
    from paper_2511_12376_b200 import quantizer as Q
    n, block, m = 1 << 30, 1 << 20, 16
    g = torch.Generator(device=dev).manual_seed(7 if dist == "adam_m" else 8)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    if dist == "adam_v":
        x.mul_(x)
    dq = Q.cluster_encode_device(x, m, block)
    out = Q.cluster_dequantize_device(dq)
    tabs = dq.host_tables()
    assert len(tabs) == 1024
    xh = x.cpu().numpy()
    del x
    full = list(range(0, 1024, 16)) + [1023]       # 65 spread blocks
    res = PO.blockwise(xh, block, m, full=full, deq=full)
    for u, r in enumerate(res):
        _tables_equal(tabs[u], r["table"], f"block {u}")
    codes = dq.codes.cpu().numpy()
    labels = dq.labels.cpu().numpy()
    outh = out.cpu().numpy()
    for u in full:
        s = u * block
        assert np.array_equal(codes[s:s + block], res[u]["codes"]), f"codes block {u}"
        assert np.array_equal(labels[s // 2:(s + block) // 2], res[u]["packed"]), f"labels {u}"
        assert np.array_equal(outh[s:s + block].view(np.uint32),
                              res[u]["deq"].view(np.uint32)), f"dequantized block {u}"


@pytest.mark.parametrize("shape,dist", [((32000, 8192), "adam_v"), ((4096, 11008), "adam_m")])
def test_per_tensor_c3_c4_units_vs_oracle(dev, shape, dist):
    import torch
    from paper_2511_12376_b200 import quantizer as Q
    n = shape[0] * shape[1]
    g = torch.Generator(device=dev).manual_seed(n % 1000)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    if dist == "adam_v":
        x.mul_(x)
    dq = Q.cluster_encode_device(x, 16, 0)
    (tab,) = dq.host_tables()
    xh = x.cpu().numpy()
    del x
    ora = PO.cluster_fit(xh, 16)
    _tables_equal(tab, ora, f"{shape}")
    packed, codes, _ = PO.cluster_quantize(xh, ora)
    assert np.array_equal(dq.codes.cpu().numpy(), codes)
    assert np.array_equal(dq.labels.cpu().numpy(), packed)


@pytest.mark.parametrize("p", [0.001, 0.01, 0.0625, 0.25])
def test_c1_full_size_vs_oracle(dev, p):
    import torch
    import bench
    from paper_2511_12376_b200 import bitmask as B
    n = 1 << 30
    base, cur, k = bench.make_c1(n, p, 11, dev)
    d = B.encode_delta_device(base, cur)
    assert d.n_c == k
    out = B.decode_delta_device(base, d.mask, d.payload, d.n_c)
    assert torch.equal(out, cur)
    del out
    bh = base.cpu().numpy().view(np.uint16)
    ch = cur.cpu().numpy().view(np.uint16)
    del base, cur
    mask, payload, n_c = PO.delta_encode(bh, ch)
    assert n_c == k
    assert np.array_equal(d.mask.cpu().numpy(), mask)
    assert np.array_equal(d.payload.cpu().numpy().view(np.uint16), payload)
