"""Template engine parity (reference anchors, exact strings) and the new
`cuda` target: a LEGO-instantiated .cu template compiles for sm_100a."""

import pytest

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import runtime as R
from paper_2505_08091_b200.template import instantiate, parse_manifest, parse_template

MANIFEST = """[layouts]
Blk = GroupBy([2,2]).OrderBy(Col(2,2))
Axis = TileBy([2],[4]).OrderBy(Row(8))
Data = GroupBy([8,8]).OrderBy(Row(8,8))

[vars]
pid in [0, 4)
pid_m in [0, 2)
pid_n in [0, 2)
k in [0, 2)
i in [0, 8)
j in [0, 8)
idx_m vec in [0, 8)
idx_k vec in [0, 8)

[target]
python
"""


def test_reference_exact_strings():
    # test_template.py:202-208, :243-249, :257-264 of the reference
    m = parse_manifest(MANIFEST)
    assert instantiate(parse_template("{{ Data[i, j] }}"), m) == "i*8 + j"
    assert instantiate(parse_template("{{ Blk.inv(pid) }}"), m) == "pid % 2, pid // 2"
    tm = parse_manifest(MANIFEST.replace("python", "triton"))
    out = instantiate(parse_template("{{ Data[0:4, :] }}"), tm)
    assert out == "(tl.arange(0, 4))[:, None]*8 + (tl.arange(0, 8))[None, :]"


def test_source_roundtrip_and_errors():
    src = "a\n {{ A[i,:] }} mid {{  j*2 }}\nend"
    assert parse_template(src).source() == src
    with pytest.raises(L.UnterminatedPlaceholder) as err:
        parse_template("line one\nx = {{ A.apply(i)")
    assert err.value.line == 2
    with pytest.raises(L.PlaceholderSyntax):
        parse_template("{{ A.frob(i) }}")
    m = parse_manifest(MANIFEST)
    with pytest.raises(L.UnknownLayout):
        instantiate(parse_template("{{ Nope[i, j] }}"), m)
    with pytest.raises(L.UnknownVariable):
        instantiate(parse_template("{{ Data[q, j] }}"), m)


CUDA_TEMPLATE = """
extern "C" __global__ void lego_tiled_copy(const float* __restrict__ src, float* __restrict__ dst) {
    const long long pid = blockIdx.x;
    const long long t = threadIdx.x;
    const long long i = {{ Rows[pid, t] }};
    const long long j = {{ Cols[pid, t] }};
    dst[{{ Tiled[i, j] }}] = src[{{ Data[i, j] }}];
}
"""

CUDA_MANIFEST = """[layouts]
Rows = GroupBy([16384],[256]).OrderBy(RegP([16384,256],[1,2]))
Cols = GroupBy([16384],[256]).OrderBy(RegP([16384,256],[1,2]))
Data = GroupBy([2048,2048]).OrderBy(Row(2048,2048))
Tiled = GroupBy([2048,2048]).OrderBy(RegP([64,32,64,32],[1,3,2,4]))

[vars]
pid in [0, 16384)
t in [0, 256)
i in [0, 2048)
j in [0, 2048)

[target]
cuda
"""


def test_cuda_target_template_compiles_for_sm100a():
    m = parse_manifest(CUDA_MANIFEST)
    src = instantiate(parse_template(CUDA_TEMPLATE), m)
    assert "{{" not in src and "lego_fdiv" not in src     # all operands provably >= 0
    assert "/ 32*65536" in src.replace("(", "").replace(")", "") or "i / 32" in src
    helpers = open(R.os.path.join(R.PKG, "csrc", "lego_index.cuh")).read()
    cubin = R.compile_cubin(helpers + src)
    assert cubin[:4] == b"\x7fELF"


def test_cuda_profile_floor_helpers_for_signed_operands():
    x = L.Var("x", L.VarRange(-8, 8))
    assert L.emit_expr(x // 4, L.CUDA_PROFILE) == "lego_fdiv(x, 4)"
    assert L.emit_expr(x % 4, L.CUDA_PROFILE) == "lego_fmod(x, 4)"
    y = L.Var("y", L.VarRange(0, 8))
    assert L.emit_expr(y // 4, L.CUDA_PROFILE) == "y / 4"
    assert L.emit_expr(L.isqrt(y), L.CUDA_PROFILE) == "lego_isqrt(y)"


def test_cuda_template_with_antidiag_inverse_compiles():
    """The antidiag inverse (isqrt, selects) spliced into a .cu template."""
    m = parse_manifest("[layouts]\nAD = GroupBy([64,64]).OrderBy(GenP([64,64], antidiag))\n"
                       "[vars]\nf in [0, 4096)\n[target]\ncuda\n")
    first, second = _split_top_level(instantiate(parse_template("{{ AD.inv(f) }}"), m))
    src = ('extern "C" __global__ void lego_antidiag_inv(long long* out) {\n'
           '    const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;\n'
           f'    const long long i = {first};\n    const long long j = {second};\n'
           '    out[f] = i * 64 + j;\n}\n')
    helpers = open(R.os.path.join(R.PKG, "csrc", "lego_index.cuh")).read()
    assert "lego_isqrt" in src
    assert R.compile_cubin(helpers + src)[:4] == b"\x7fELF"


def _split_top_level(text):
    depth = 0
    for k, ch in enumerate(text):
        depth += ch in "(["
        depth -= ch in ")]"
        if ch == "," and depth == 0:
            return text[:k].strip(), text[k + 1:].strip()
    raise AssertionError(text)


USER_TEMPLATE = """
// a user kernel written against LEGO layouts: copy a row-major 256 x 256
// matrix into the 32 x 32 tiled layout, and record the anti-diagonal inverse
extern "C" __global__ void lego_tpl_tile(const float* __restrict__ src, float* __restrict__ dst) {
    const long long i = blockIdx.x;
    const long long j = threadIdx.x;
    dst[{{ Tiled[i, j] }}] = src[{{ Data[i, j] }}];
}
extern "C" __global__ void lego_tpl_antidiag_inv(long long* __restrict__ out) {
    const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long ij[2] = { {{ AD.inv(f) }} };
    out[f] = ij[0] * 64 + ij[1];
}
"""

USER_MANIFEST = """[layouts]
Data = GroupBy([256,256]).OrderBy(Row(256,256))
Tiled = GroupBy([256,256]).OrderBy(RegP([8,32,8,32],[1,3,2,4]))
AD = GroupBy([64,64]).OrderBy(GenP([64,64], antidiag))

[vars]
i in [0, 256)
j in [0, 256)
f in [0, 4096)

[target]
cuda
"""


@pytest.mark.gpu
def test_instantiated_cuda_template_runs():
    """a .cu template instantiated with the cuda target is
    compiled, launched, and its output checked against the C oracle."""
    import ctypes

    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_2505_08091_b200 import kernels as K
    mod = K.compile_template(USER_TEMPLATE, USER_MANIFEST)
    src = torch.arange(256 * 256, dtype=torch.float32, device="cuda")
    dst = torch.empty_like(src)
    mod.launch("lego_tpl_tile", (256,), (256,), [ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr())])
    spec = O.parse("GroupBy([256,256]).OrderBy(RegP([8,32,8,32],[1,3,2,4]))")
    want = O.remap(src.cpu().numpy(), None, spec)
    assert np.array_equal(dst.cpu().numpy(), want)
    out = torch.empty(4096, dtype=torch.int64, device="cuda")
    mod.launch("lego_tpl_antidiag_inv", (16,), (256,), [ctypes.c_void_p(out.data_ptr())])
    assert np.array_equal(out.cpu().numpy(), O.inv_range(O.parse("GroupBy([64,64]).OrderBy(GenP([64,64], antidiag))")))


def test_user_template_compiles():
    from paper_2505_08091_b200 import kernels as K
    from paper_2505_08091_b200.template import instantiate, parse_manifest, parse_template
    src = instantiate(parse_template(USER_TEMPLATE), parse_manifest(USER_MANIFEST))
    assert "{{" not in src and "lego_isqrt" in src
    helpers = open(R.os.path.join(R.PKG, "csrc", "lego_index.cuh")).read()
    assert R.compile_cubin(helpers + "\n" + src)[:4] == b"\x7fELF"
    assert K.compile_template  # loading needs a GPU (test_instantiated_cuda_template_runs)
