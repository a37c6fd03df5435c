"""PLY checkpoint loading (ply.hpp, ply.cpp).

CPU tests: the host reader behind sgs_ply_read / load_scene is compared with the
reference's own load_ply (oracle/_ref) on files the reference writes with save_ply,
on hand-edited variants (ASCII, permuted columns, ignored normals, CRLF, obj_info,
sidecar) and on every error case, message for message. The committed fixtures in
tests/golden/ply/ pin the reader without the reference (the GPU box has none).
GPU tests: the device loader (rows -> planes on the GPU) produces the same scene
blob, byte for byte, as uploading the host-read parameters.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2501_00342_b200 as sg
from oracle_lib import FlatScene

GOLDEN_PLY = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ply")

STATUS_OF = {sg.InvalidArgumentError: 1, sg.NumericError: 2, sg.IoError: 7, sg.FormatError: 8}


def ours(path):
    """(0, Scene) or (status, message) from our host reader."""
    try:
        return 0, sg.load_scene(str(path))
    except (sg.InvalidArgumentError, sg.NumericError, sg.IoError, sg.FormatError) as e:
        return STATUS_OF[type(e)], str(e)


def assert_same(ref, path):
    rc_r, r = ref.load_ply(path)
    rc_o, o = ours(path)
    assert rc_o == rc_r, (rc_o, o, rc_r, r)
    if rc_r != 0:
        assert o == r  # the reference's message
        return None
    assert o.params.shape[0] == r.n
    if r.n:
        assert o.kind == r.kind and o.sh_degree == r.degree
        assert np.array_equal(o.params, r.params)  # bit for bit
    assert np.array_equal(o.shared_axes, r.axes) and np.array_equal(o.background, r.background)
    return o


# -- helpers to rewrite PLY files ---------------------------------------------------
def read_ply(path):
    data = open(path, "rb").read()
    end = data.index(b"end_header\n") + len(b"end_header\n")
    header = data[:end].decode().split("\n")[:-1]
    props = [ln.split()[2] for ln in header if ln.startswith("property")]
    count = int([ln for ln in header if ln.startswith("element")][0].split()[2])
    rows = np.frombuffer(data[end:], dtype="<f4").reshape(count, len(props))
    return header, props, rows


def write_ply(path, header_lines, props, rows, binary=True, newline="\n"):
    out = []
    for ln in header_lines:
        if ln.startswith("property") or ln.startswith("end_header") or ln.startswith("element"):
            continue
        if ln.startswith("format"):
            ln = "format binary_little_endian 1.0" if binary else "format ascii 1.0"
        out.append(ln)
    out.append(f"element vertex {rows.shape[0]}")
    out += [f"property float {p}" for p in props]
    out.append("end_header")
    with open(path, "wb") as f:
        f.write((newline.join(out) + newline).encode())
        if binary:
            f.write(np.ascontiguousarray(rows, dtype="<f4").tobytes())
        else:
            for row in rows:
                f.write((" ".join("%.9g" % v for v in row) + newline).encode())


SCENES = [("sh", 3, 0), ("sh", 1, 0), ("sh", 0, 0), ("sg1", 0, 1), ("sg3", 0, 1), ("mixed", 2, 1)]


@pytest.fixture
def saved(ref, tmp_path):
    """The reference's save_ply of a synthetic scene of every model."""
    out = {}
    for kind, deg, layout in SCENES:
        s = ref.synth(64, 4242, kind, deg, (-4.5, -2.5))
        if kind != "sh":
            s.background = np.array([0.25, 0.5, 0.125])
        path = tmp_path / f"{kind}{deg}.ply"
        assert ref.save_ply(s, path, layout) == 0, ref.err()
        out[(kind, deg)] = path
    return out


def test_reference_saved_files_load_identically(ref, saved):
    for (kind, deg), path in saved.items():
        o = assert_same(ref, path)
        assert o.kind == kind and o.sh_degree == (3 if kind == "sh" else deg)
        info = sg.ply_info(str(path))
        assert info.count == 64 and info.binary == 1
        assert info.layout == (0 if kind == "sh" else 1)


def test_ascii_crlf_permuted_columns_and_normals(ref, saved, tmp_path):
    rng = np.random.default_rng(5)
    for (kind, deg), path in saved.items():
        header, props, rows = read_ply(path)
        perm = rng.permutation(len(props))
        props2 = [props[i] for i in perm]
        rows2 = rows[:, perm]
        if kind == "sh":  # Reference3DGS tolerates (and ignores) normals
            props2 = props2 + ["nx", "ny", "nz"]
            rows2 = np.concatenate([rows2, rng.standard_normal((rows.shape[0], 3)).astype("<f4")], 1)
        header2 = header[:2] + ["obj_info written by a test"] + header[2:]
        for binary, nl in ((True, "\n"), (False, "\n"), (False, "\r\n")):
            p = tmp_path / f"v_{kind}{deg}_{int(binary)}_{len(nl)}.ply"
            write_ply(p, header2, props2, rows2, binary=binary, newline=nl)
            assert_same(ref, p)


def test_meta_sidecar(ref, saved, tmp_path):
    for (kind, deg), path in saved.items():
        p = tmp_path / f"side_{kind}{deg}.ply"
        p.write_bytes(path.read_bytes())
        c, s = np.cos(0.3), np.sin(0.3)
        axes = [c, -s, 0, s, c, 0, 0, 0, 1]
        (tmp_path / (p.name + ".meta")).write_text(
            "axes=" + " ".join(repr(v) for v in axes) + "\nbackground=0.1 0.2 0.3\nignored line\n")
        o = assert_same(ref, p)
        assert np.allclose(o.background, [0.1, 0.2, 0.3])


def test_empty_checkpoints(ref, saved, tmp_path):
    s = FlatScene("sh", 3, np.zeros((0, 11)), np.eye(3), np.zeros(3))
    p = tmp_path / "empty_reference.ply"
    assert ref.save_ply(s, p, 0) == 0, ref.err()
    assert_same(ref, p)
    # save_ply cannot write an empty SG scene (its kind is unknown): edit saved files
    for kind in (("sg1", 0), ("sg3", 0), ("mixed", 2)):
        header, props, rows = read_ply(saved[kind])
        p = tmp_path / f"empty_{kind[0]}.ply"
        write_ply(p, header, props, rows[:0])
        assert_same(ref, p)


def test_error_cases_match_reference(ref, saved, tmp_path):
    sh, mixed, sg3 = saved[("sh", 3)], saved[("mixed", 2)], saved[("sg3", 0)]
    cases = []
    cases.append(tmp_path / "does_not_exist.ply")
    (tmp_path / "empty.ply").write_bytes(b"")
    cases.append(tmp_path / "empty.ply")
    (tmp_path / "notply.ply").write_bytes(b"PLY\nformat ascii 1.0\n")
    cases.append(tmp_path / "notply.ply")
    (tmp_path / "trunc_header.ply").write_bytes(b"ply\nformat ascii 1.0\nelement vertex 1\n")
    cases.append(tmp_path / "trunc_header.ply")
    (tmp_path / "noformat.ply").write_bytes(b"ply\nelement vertex 0\nend_header\n")
    cases.append(tmp_path / "noformat.ply")

    for name, src, old, new in [
        ("bigendian", sh, b"binary_little_endian", b"binary_big_endian"),
        ("face", sh, b"element vertex", b"element face"),
        ("double", sh, b"property float x", b"property double x"),
        ("badline", sh, b"format", b"bogus line\nformat"),
        ("twovertex", sh, b"end_header", b"element vertex 0\nend_header"),
        ("propfirst", sh, b"element vertex", b"property float q\nelement vertex"),
        ("nomodel", mixed, b"comment sg_model mixed", b"comment other mixed"),
        ("shmodel", mixed, b"comment sg_model mixed", b"comment sg_model sh"),
        ("badmodel", mixed, b"comment sg_model mixed", b"comment sg_model foo"),
        ("badaxes", sg3, b"comment sg_axes", b"comment sg_axes x"),
        ("skewaxes", sg3, b"comment sg_axes 1", b"comment sg_axes 1.5"),
        ("badbg", sg3, b"comment sg_background", b"comment sg_background x"),
        ("unknownprop", sh, b"property float rot_3", b"property float rot_3\nproperty float extra"),
        ("dupprop", sh, b"property float rot_3", b"property float rot_2"),
        ("both", sh, b"property float rot_3", b"property float rot_3\nproperty float sg_alpha_0_0"),
        ("neither", sh, b"property float f_rest_0\n", b"property float q_rest_0\n"),
    ]:
        p = tmp_path / f"{name}.ply"
        p.write_bytes(src.read_bytes().replace(old, new, 1))
        cases.append(p)
    # truncated payloads (binary and ASCII) and a missing property
    data = sh.read_bytes()
    (tmp_path / "trunc.ply").write_bytes(data[:-10])
    cases.append(tmp_path / "trunc.ply")
    header, props, rows = read_ply(sh)
    write_ply(tmp_path / "ascii_trunc.ply", header, props, rows, binary=False)
    txt = (tmp_path / "ascii_trunc.ply").read_text()
    (tmp_path / "ascii_trunc.ply").write_text(txt[: len(txt) - 40])
    cases.append(tmp_path / "ascii_trunc.ply")
    write_ply(tmp_path / "missing.ply", header, props[:-1], rows[:, :-1])
    cases.append(tmp_path / "missing.ply")
    for p in cases:
        rc_r, _ = ref.load_ply(p)
        assert rc_r != 0, p
        assert_same(ref, p)


def test_crafted_vertex_counts_fail_safely(tmp_path):
    """A header whose vertex count times the property count wraps 64 bits (or just
    exceeds the file) must fail as a truncated payload before anything is sized from
    it -- not overrun a buffer sized from the wrapped product."""
    props = [f"p{i}" for i in range(16)]
    body = np.zeros((1, 16), dtype="<f4").tobytes()
    for count in (2 ** 60 + 1, 2 ** 62, 2 ** 64 - 1, 2):  # 16 * (2^60 + 1) == 16 (mod 2^64)
        for binary in (True, False):
            p = tmp_path / f"crafted_{count}_{int(binary)}.ply"
            hdr = ["ply", "format binary_little_endian 1.0" if binary else "format ascii 1.0",
                   f"element vertex {count}"] + [f"property float {q}" for q in props] + ["end_header"]
            payload = body if binary else (" ".join(["0"] * 16) + "\n").encode()
            p.write_bytes(("\n".join(hdr) + "\n").encode() + payload)
            for call in (sg.load_scene, sg.ply_info):
                with pytest.raises(sg.IoError, match="truncated"):
                    call(str(p))


def test_golden_ply_fixtures():
    """Without the reference: the committed files and their reference-loaded params."""
    idx = np.load(os.path.join(GOLDEN_PLY, "expected.npz"))
    names = [k[:-7] for k in idx.files if k.endswith(".params")]
    assert names
    for name in names:
        s = sg.load_scene(os.path.join(GOLDEN_PLY, name))
        assert np.array_equal(s.params, idx[name + ".params"])
        assert np.array_equal(s.shared_axes.reshape(9), idx[name + ".axes"])
        assert np.array_equal(s.background, idx[name + ".bg"])
        assert s.kind == str(idx[name + ".kind"]) and s.sh_degree == int(idx[name + ".deg"])


@pytest.mark.gpu
def test_device_loader_matches_host_upload():
    """sgs_scene_load_ply (rows scattered on the GPU) == sgs_scene_upload of the
    host-read parameters: identical blob bytes and identical renders."""
    import torch

    r = sg.Renderer(0)
    cams = sg.orbit_cameras(2, 160, 120, 3.0, 144.0)
    idx = np.load(os.path.join(GOLDEN_PLY, "expected.npz"))
    for name in [k[:-7] for k in idx.files if k.endswith(".params")]:
        path = os.path.join(GOLDEN_PLY, name)
        a = r.load_ply(path)
        b = r.upload(sg.load_scene(path))
        try:
            ma, mb = a.meta, b.meta
            assert bytes(ma) == bytes(mb)
            pa, na = a.blob()
            pb, nb = b.blob()
            assert na == nb
            assert torch.equal(_device_bytes(pa, na), _device_bytes(pb, nb)), name
            if ma.count:
                ra = r.render_batch(a, cams)
                rb = r.render_batch(b, cams)
                assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
        finally:
            a.free()
            b.free()


class _DevView:
    """A raw device allocation seen by torch through __cuda_array_interface__."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3}


def _device_bytes(ptr, n):
    import torch

    torch.cuda.synchronize()
    return torch.as_tensor(_DevView(ptr, n), device="cuda").clone()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,deg", [("sh", 3), ("sg1", 0), ("sg3", 0), ("mixed", 2)])
def test_f32_row_upload_matches_host_packing(kind, deg):
    """sgs_scene_upload of an SGS_F32 description (rows scattered into the planes on
    the device, the drop-in render's path) == the float64 description packed on the
    host: identical blob bytes."""
    import torch

    r = sg.Renderer(0)
    s = sg.synth_scene(20_000, kind, 77, sh_degree=deg)
    if kind == "sg1":  # un-normalised (still f32-exact) lobe axes: the FP64 normalisation runs on the device
        s.params[:, 11 + 7:11 + 10] *= 2.0
    a, b = r.upload(s), r.upload(s, f32=True)
    try:
        assert bytes(a.meta) == bytes(b.meta)
        pa, na = a.blob()
        pb, nb = b.blob()
        assert torch.equal(_device_bytes(pa, na), _device_bytes(pb, nb))
    finally:
        a.free()
        b.free()
