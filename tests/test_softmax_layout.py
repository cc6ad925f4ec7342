"""The softmax's thread/data layout is a LEGO layout and its offsets are
generated from it (the paper's softmax: index ops 4 -> 0).

CPU: ``apply_symbolic`` of ``GroupBy([rows],[cols/4T],[T],[4]).OrderBy(Row(rows, cols))``
simplifies to ``row*cols + it*4T + tid*4 + v``, and the generated program
source's ``gen::vec_of`` is that offset over 4.
GPU: the offsets the generated program's kernel accesses (dumped by
``lego_softmax_offsets`` from the same device function) equal the layout's
``apply`` computed by the generated index-map kernel; the program's results
are within 1e-5 (max relative) of float64.
"""

import pytest

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K

T = K.SOFTMAX_THREADS


@pytest.mark.parametrize("cols", [1024, 4096, 8192, 16384])
def test_layout_offset_is_row_major(cols):
    rows = 8
    lay = K.softmax_layout(cols, rows=rows)
    row, it, tid, v = L.index_vars(["row", "it", "tid", "v"], lay.dims)
    off = L.apply_symbolic(lay, (row, it, tid, v))
    want = row * cols + it * (4 * T) + tid * 4 + v
    assert L.simplify(off - want) == L.IntConst(0)
    assert L.op_count(off) <= L.op_count(L.simplify(want))


def test_generated_source_uses_the_layout():
    src, info = K.softmax_source(8192)
    assert "#define SM_GEN 1" in src and "vec_of" in src
    assert info.kind == 7 and info.n == 8192 and info.units == (1 << 36) // 8192
    from paper_2505_08091_b200 import runtime as R
    assert len(R.compile_cubin(src)) > 1000


def test_program_path_selection():
    assert K.softmax_generated(8192) and K.softmax_generated(1024) and K.softmax_generated(16384)
    assert not K.softmax_generated(1000) and not K.softmax_generated(32768) and not K.softmax_generated(2000)


@pytest.mark.gpu
@pytest.mark.parametrize("cols", [1024, 4096, 8192, 16384])
def test_device_offsets_are_the_layout(cols):
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import runtime as R
    rows = 3
    prog = K.softmax_program(cols)
    its = cols // (4 * T)
    got = torch.empty(rows * its * T, dtype=torch.int64, device="cuda")
    R.check(R.lib().lego_softmax_offsets(prog.handle, got.data_ptr(), rows, R.stream_handle(None)))
    pos = K.apply_map(K.softmax_layout(cols), dtype=torch.int64, count=rows * cols)
    want = pos.view(rows, its, T, 4)[..., 0].reshape(-1)
    assert torch.equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols", [(8192, 8192), (3, 1024), (17, 16384), (64, 2048)])
def test_generated_softmax_numerics(rows, cols):
    torch = pytest.importorskip("torch")
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(rows, cols, device="cuda", generator=g) * 4
    y = K.softmax(x)
    ref = torch.softmax(x.double(), dim=-1)
    rel = ((y.double() - ref).abs() / ref.abs().clamp_min(1e-30)).max().item()
    assert rel <= 1e-5, rel
