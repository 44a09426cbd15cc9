"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/mcs.h
declares, and behaves on host-only logic (no compute calls without a GPU)."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import paper_2504_18056_b200 as mcs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = mcs.load()
    names = mcs.header_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n


def test_config_defaults_follow_the_paper_readings():
    cfg = mcs.default_config()
    assert cfg.abi_version == mcs.ABI_VERSION
    assert cfg.neighbor_count == 3
    assert cfg.loop_recency_gap == 10                   # R5
    assert cfg.voxel_resolution == 0.5                  # R10
    assert cfg.gn_slots == 0                            # R4 (Fig.3)
    assert cfg.damping_rel == 1e-6 and cfg.step_clamp == 1.0   # R11
    assert cfg.unmatched_penalty == 0.0                 # R8
    assert cfg.loglik_rel_floor == math.log(1e-16)      # P:190, R17
    assert cfg.posterior_floor == 1e-8
    assert cfg.world_size == 1 and cfg.rank == 0
    assert cfg.kf_table_mib == 64 and cfg.graph_replay == 1 and cfg.point_splits == 0


def test_state_bytes_linear_in_keyframes_and_paper_memory_figure():
    """per-particle memory grows only with the keyframe count (clouds are shared);
    100,000 particles x 100 keyframes of 4x4 fp32 poses = 610.35 MiB."""
    b = [mcs.state_bytes_per_particle(k) for k in range(0, 201)]
    d = np.diff(b)
    assert np.all(d == 48)                              # one 3x4 fp32 pose per keyframe
    assert b[0] == 48 + 8                               # T_t + fp64 L
    assert 100_000 * 100 * 64 / 2**20 == pytest.approx(610.3515625, abs=0)
    ours = 100_000 * (mcs.state_bytes_per_particle(100)) / 2**20
    assert ours < 610.36                                # 3x4 storage fits the paper's budget


def test_create_validates_before_touching_the_device():
    bad = [dict(capacity_particles=0), dict(neighbor_count=5), dict(voxel_resolution=0.3),
           dict(abi_version=99), dict(world_size=2, rank=1), dict(capacity_particles=(1 << 21) + 1),
           dict(corr_mode=1, nn_radius=0.0), dict(corr_mode=1, nn_radius=1.0), dict(corr_mode=3),
           dict(clone_split=2),
           dict(allocator=mcs.Allocator(mcs.mcs.ALLOC_FN(lambda n, s, u: None),
                                        mcs.mcs.FREE_FN(), None))]
    for kw in bad:
        base = dict(capacity_particles=100, capacity_keyframes=4, capacity_scan_points=64)
        base.update(kw)
        with pytest.raises(mcs.MCSError) as ei:
            mcs.Context(**base)
        assert ei.value.status in (1, 5), (kw, ei.value)


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mcs.MCSError) as ei:
        mcs.Context(100, 4, 64)
    assert ei.value.status == 3  # MCS_E_CUDA, message from the runtime


def test_unpack_h21_roundtrip():
    g = np.random.default_rng(0)
    A = g.normal(size=(5, 6, 6))
    A = A + A.transpose(0, 2, 1)
    iu = np.triu_indices(6)
    h21 = A[:, iu[0], iu[1]]
    np.testing.assert_array_equal(mcs.unpack_h21(h21), A)


def test_config_mirror_matches_the_header():
    """The ctypes mirror of mcs_config has the header's fields in the header's order and the
    library's size (a mismatch once let mcs_config_default write past the Python struct)."""
    import ctypes as C
    import re
    src = open(os.path.join(ROOT, "include", "mcs.h")).read()
    body = src[src.index("typedef struct mcs_config {"):src.index("} mcs_config;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split("{", 1)[1].split(";"):
        decl = decl.strip()
        if not decl:
            continue
        for part in decl.split(","):
            names.append(re.findall(r"[A-Za-z_]\w*", part)[-1])
    assert [f for f, _ in mcs.Config._fields_] == names
    assert C.sizeof(mcs.Config) == mcs.load().mcs_config_size()


def _header_fields(closing):
    """Member names of the struct typedef that ends with `closing` in include/mcs.h."""
    import re
    src = open(os.path.join(ROOT, "include", "mcs.h")).read()
    end = src.index(closing)
    body = src[src.rindex("typedef struct", 0, end):end]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S).split("{", 1)[1]
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        if "(" in decl:  # function pointer: int (*name)(...)
            names.append(re.search(r"\(\s*\*\s*(\w+)\s*\)", decl).group(1))
            continue
        for part in decl.split(","):
            names.append(re.findall(r"[A-Za-z_]\w*", part)[-1])
    return names


def test_other_struct_mirrors_match_the_header():
    import ctypes as C
    assert [f for f, _ in mcs.mcs.UpdateOut._fields_] == _header_fields("} mcs_update_out;")
    assert [f for f, _ in mcs.mcs.Transport._fields_] == _header_fields("} mcs_transport;")
    assert [f for f, _ in mcs.mcs.Allocator._fields_] == _header_fields("} mcs_allocator;")
    assert [f for f, _ in mcs.Config._fields_] == _header_fields("} mcs_config;")
    # all pointer-sized members
    assert C.sizeof(mcs.mcs.UpdateOut) == 8 * len(mcs.mcs.UpdateOut._fields_)
    assert C.sizeof(mcs.mcs.Transport) == 32 and C.sizeof(mcs.mcs.Allocator) == 24
