"""The HBM-bound reference kernels on their vector and scalar paths:
gen_filter_checksum (checksum.hpp:75-90) and ic_batch_checksum (:350-362) as
column sums of an int8 matrix, and the standalone epilog (convolution.hpp:353-387)
-- bit-exact against the C oracle on aligned, ragged and extreme inputs."""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Oracle
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


@pytest.mark.parametrize("kcrs", [(64, 64, 3, 3), (512, 512, 3, 3), (3, 5, 3, 3), (300, 3, 3, 3), (1, 16, 1, 1),
                                  (7, 1, 1, 1), (1000, 16, 1, 1), (40000, 16, 1, 1), (2048, 512, 1, 1)])
@pytest.mark.parametrize("extreme", [False, True])
@pytest.mark.parametrize("kernel", ["0", "3", "4"], ids=["auto", "tall", "cluster"])
def test_filter_checksum(ora, kcrs, extreme, kernel, monkeypatch):
    monkeypatch.setenv("ABED_COLSUM_KERNEL", kernel)
    g = torch.Generator().manual_seed(sum(kcrs))
    f = torch.full(kcrs, -128, dtype=torch.int8) if extreme else torch.randint(-128, 128, kcrs, dtype=torch.int8,
                                                                                generator=g)
    got = api.gen_filter_checksum(f.cuda()).cpu().numpy()
    assert np.array_equal(got, ora.gen_filter_checksum(f.numpy()))


@pytest.mark.parametrize("nchw", [(32, 64, 56, 56), (3, 5, 7, 9), (1, 16, 4, 4), (129, 8, 2, 1), (2, 3, 1, 1)])
def test_batch_checksum(nchw):
    g = torch.Generator().manual_seed(sum(nchw))
    x = torch.randint(-128, 128, nchw, dtype=torch.int8, generator=g)
    got = api.ic_batch_checksum(x.cuda()).cpu()
    assert torch.equal(got, x.to(torch.int32).sum(0, keepdim=True))


@pytest.mark.parametrize("kernel", ["1", "3", "4"], ids=["wide", "tall", "cluster"])
@pytest.mark.parametrize("nchw", [(40, 64, 56, 56), (300, 4, 32, 32), (17, 3, 100, 100), (1, 16, 16, 16),
                                  (513, 1, 4, 4)])
@pytest.mark.parametrize("fill", [None, 127, -128])
def test_batch_checksum_kernels(nchw, kernel, fill, monkeypatch):
    """The three 16-byte-vector column-sum kernels (4096-column tiles reading
    whole pages per row, 32-column tiles over all rows, 512-column tiles with
    row-split clusters), forced by ABED_COLSUM_KERNEL, with more than 256 rows per
    thread lane (the 16-bit flush) and the extreme values of both signs."""
    monkeypatch.setenv("ABED_COLSUM_KERNEL", kernel)
    g = torch.Generator().manual_seed(sum(nchw))
    x = torch.full(nchw, fill, dtype=torch.int8) if fill is not None else \
        torch.randint(-128, 128, nchw, dtype=torch.int8, generator=g)
    got = api.ic_batch_checksum(x.cuda()).cpu()
    assert torch.equal(got, x.to(torch.int32).sum(0, keepdim=True))


@pytest.mark.parametrize("nkpq", [(2, 64, 56, 56), (1, 3, 5, 7), (2, 16, 4, 4), (1, 8, 3, 16)])
@pytest.mark.parametrize("relu", [True, False])
@pytest.mark.parametrize("kind", [abi.I8, abi.F32])
def test_epilog(ora, nkpq, relu, kind):
    g = torch.Generator().manual_seed(sum(nkpq) + relu)
    acc = torch.randint(-40000, 40000, nkpq, dtype=torch.int32, generator=g)
    acc.view(-1)[:4] = torch.tensor([0, 2**31 - 1, -2**31, -21774], dtype=torch.int32)
    bias = np.linspace(-3.0, 3.0, nkpq[1]).astype(np.float32)
    scale = 0.0123
    got = api.epilog(acc.cuda(), scale, bias, relu, kind).cpu().numpy()
    want = ora.epilog(acc.numpy(), scale, bias, relu=relu, out_f32=kind == abi.F32)
    assert np.array_equal(got.view(np.uint8), np.asarray(want).view(np.uint8))


@pytest.mark.parametrize("nv", ["1", "2", "4", "8"])
@pytest.mark.parametrize("kcrs", [(512, 512, 3, 3), (300, 3, 3, 3), (1000, 16, 1, 1), (70, 9, 5, 5)])
def test_filter_checksum_tall_widths(ora, kcrs, nv, monkeypatch):
    """The tall column-sum kernel at every column width per CTA (16 * NV)."""
    monkeypatch.setenv("ABED_COLSUM_KERNEL", "3")
    monkeypatch.setenv("ABED_COLSUM_TALL_NV", nv)
    g = torch.Generator().manual_seed(sum(kcrs) + int(nv))
    f = torch.randint(-128, 128, kcrs, dtype=torch.int8, generator=g)
    got = api.gen_filter_checksum(f.cuda()).cpu().numpy()
    assert np.array_equal(got, ora.gen_filter_checksum(f.numpy()))
