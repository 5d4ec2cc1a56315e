"""Deterministic corpus of mesh files for the load_mesh parity tests.

Hand-written edge cases after reference/proj/tests/test_io.cpp and
test_mesh.cpp:26-64 (unit square OBJ, ASCII PLY with extra properties, the
error sections: missing magic, quad face, wrong element order, truncated
binary payload, index range), widened to the corners of the reference
loader (mesh_io.hpp): std::istream >> double token rules, relative OBJ
indices, every PLY scalar type, list-count casts, extra elements, byte-offset
truncation, plus seeded random mutations of valid files. Expected outcomes come
from the reference itself (tests/golden/make_io_golden.py -> io_cases.json).
"""
from __future__ import annotations

import struct

import numpy as np

OBJ, PLY = 0, 1

SQUARE_OBJ = b"v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1 2 3\nf 1 3 4\n"

PLY_ASCII_HEAD = (b"ply\nformat ascii 1.0\nelement vertex 4\nproperty float x\nproperty float y\nproperty float z\n"
                  b"element face 2\nproperty list uchar int vertex_indices\nend_header\n")
SQUARE_PLY_BODY = b"0 0 0\n1 0 0\n1 1 0\n0 1 0\n3 0 1 2\n3 0 2 3\n"

_PACK = {"char": "b", "int8": "b", "uchar": "B", "uint8": "B", "short": "h", "int16": "h", "ushort": "H",
         "uint16": "H", "int": "i", "int32": "i", "uint": "I", "uint32": "I", "float": "f", "float32": "f",
         "double": "d", "float64": "d"}


def grid(nx: int, ny: int, jitter: float = 0.0, seed: int = 0):
    """(positions [V,3], faces [F,3]) of a triangulated nx x ny grid."""
    rng = np.random.RandomState(seed)
    xs, ys = np.meshgrid(np.arange(nx + 1, dtype=np.float64), np.arange(ny + 1, dtype=np.float64), indexing="xy")
    P = np.stack([xs.ravel() / nx, ys.ravel() / ny, np.zeros(xs.size)], axis=1)
    if jitter:
        P[:, 2] = jitter * rng.standard_normal(P.shape[0])
    F = []
    for j in range(ny):
        for i in range(nx):
            a = j * (nx + 1) + i
            b, c, d = a + 1, a + nx + 2, a + nx + 1
            F += [[a, b, c], [a, c, d]] if (i + j) % 2 == 0 else [[a, b, d], [b, c, d]]
    return P, np.asarray(F, dtype=np.int32)


def obj_text(P, F, fmt="%.17g") -> bytes:
    out = [("v " + " ".join(fmt % x for x in p) + "\n") for p in P]
    out += ["f %d %d %d\n" % (a + 1, b + 1, c + 1) for a, b, c in F]
    return "".join(out).encode()


def ply_ascii(P, F, vprops=("x", "y", "z"), extra=b"") -> bytes:
    h = [b"ply", b"format ascii 1.0", b"element vertex %d" % len(P)]
    h += [b"property double " + p.encode() for p in vprops]
    h += [b"element face %d" % len(F), b"property list uchar int vertex_indices", b"end_header"]
    body = [(" ".join("%.17g" % x for x in p)).encode() for p in P]
    body += [b"3 %d %d %d" % tuple(f) for f in F]
    return b"\n".join(h) + b"\n" + b"\n".join(body) + b"\n" + extra


def ply_binary(vprops, vrows, fprops, frows, extra_elements=(), fmt=b"binary_little_endian") -> bytes:
    """vprops: [(type, name)]; fprops: [(type, name)] or [("list", ctype, vtype, name)];
    rows: tuples of values (a list property's value is a Python list)."""
    h = [b"ply", b"format " + fmt + b" 1.0", b"element vertex %d" % len(vrows)]
    for p in vprops:
        h.append(_prop_line(p))
    h.append(b"element face %d" % len(frows))
    for p in fprops:
        h.append(_prop_line(p))
    for name, props, rows in extra_elements:
        h.append(b"element %s %d" % (name.encode(), len(rows)))
        for p in props:
            h.append(_prop_line(p))
    h.append(b"end_header")
    out = b"\n".join(h) + b"\n"
    out += b"".join(_pack_row(vprops, r) for r in vrows)
    out += b"".join(_pack_row(fprops, r) for r in frows)
    for _name, props, rows in extra_elements:
        out += b"".join(_pack_row(props, r) for r in rows)
    return out


def _prop_line(p) -> bytes:
    if p[0] == "list":
        return ("property list %s %s %s" % (p[1], p[2], p[3])).encode()
    return ("property %s %s" % (p[0], p[1])).encode()


def _pack_row(props, row) -> bytes:
    out = b""
    for p, v in zip(props, row):
        if p[0] == "list":
            out += struct.pack("<" + _PACK[p[1]], len(v) if not isinstance(v, tuple) else v[0])
            vals = v if not isinstance(v, tuple) else v[1]
            out += b"".join(struct.pack("<" + _PACK[p[2]], x) for x in vals)
        else:
            out += struct.pack("<" + _PACK[p[0]], v)
    return out


def _xyz_double():
    return [("double", "x"), ("double", "y"), ("double", "z")]


def _tri_list(ctype="uchar", vtype="int"):
    return [("list", ctype, vtype, "vertex_indices")]


def square_binary(**kw) -> bytes:
    P, F = grid(1, 1)
    return ply_binary(_xyz_double(), [tuple(p) for p in P], _tri_list(), [([int(x) for x in f],) for f in F], **kw)


# ------------------------------------------------------------------ cases
def hand_cases():
    C = []
    add = lambda name, fmt, data: C.append((name, fmt, data))  # noqa: E731
    # ---- OBJ (mesh_io.hpp:39-78, test_mesh.cpp:26-64)
    add("obj_square", OBJ, SQUARE_OBJ)
    add("obj_square_crlf_tabs_comments", OBJ,
        b"# unit square\r\nv\t0 0 0\r\nv 1 0 0 \r\n\r\nv 1 1 0\r\nvn 0 0 1\r\nvt 0 0\r\n#v 9 9 9\r\nv 0 1 0\r\n"
        b"o obj\r\ng grp\r\ns off\r\nusemtl m\r\nf 1 2 3\r\nf 1 3 4")
    add("obj_slashes", OBJ, b"v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1/1/1 2/2/2 3//3\nf 1/9 3 4/4/4\n")
    add("obj_negative_indices", OBJ, b"v 0 0 0\nv 1 0 0\nv 1 1 0\nf -3 -2 -1\nv 0 1 0\nf 1 -2 -1\n")
    add("obj_w_and_extra_tokens", OBJ, b"v 0 0 0 1\nv 1 0 0 1 2 3\nv 1 1 0\nf 1 2 3\n")
    add("obj_number_forms", OBJ,
        b"v +0.5 -.5 00001.2500\nv 1e0 0E+0 -0e-0\nv 1.5e2 2.5E-1 .75\nf 1 2 3\n")
    add("obj_number_split_tokens", OBJ, b"v 1.2.3 4\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_exponent_then_digit", OBJ, b"v 1e5x 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_dangling_exponent", OBJ, b"v 0 0 0\nv 1e 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_dangling_exponent_sign", OBJ, b"v 0 0 0\nv 1.5e+ 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_hex_float", OBJ, b"v 0x1p3 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_inf", OBJ, b"v inf 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_nan", OBJ, b"v nan 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_overflow", OBJ, b"v 1e400 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_underflow", OBJ, b"v 0 0 0\nv 1 1e-400 0\nv 0 1 4.9e-324\nf 1 2 3\n")
    add("obj_long_mantissa", OBJ,
        b"v 0.1000000000000000055511151231257827021181583404541015625 0 0\n"
        b"v 1.00000000000000011102230246251565404236316680908203125 0 0.30000000000000004\n"
        b"v 0 1 123456789012345678901234567890\nf 1 2 3\n")
    add("obj_many_leading_zeros", OBJ, b"v " + b"0" * 200 + b"1.5 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_bad_vertex_short", OBJ, b"v 0 0 0\nv 1 0\nv 0 1 0\nf 1 2 3\n")
    add("obj_bad_vertex_alpha", OBJ, b"v 0 0 0\nv a b c\n")
    add("obj_sign_only", OBJ, b"v - 0 0\n")
    add("obj_dot_only", OBJ, b"v . 0 0\n")
    add("obj_quad", OBJ, b"v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1 2 3 4\n")
    add("obj_two_entry_face", OBJ, b"v 0 0 0\nv 1 0 0\nv 1 1 0\nf 1 2\n")
    add("obj_empty_face", OBJ, b"v 0 0 0\nv 1 0 0\nv 1 1 0\nf\n")
    add("obj_bad_face_entry", OBJ, b"v 0 0 0\nv 1 0 0\nv 1 1 0\nf 1 2 x\n")
    add("obj_bad_face_entry_slash_first", OBJ, b"v 0 0 0\nv 1 0 0\nv 1 1 0\nf /1 2 3\n")
    add("obj_bad_face_entry_before_count", OBJ, b"v 0 0 0\nv 1 0 0\nv 1 1 0\nf 1 2 3 4 q\n")
    add("obj_face_index_out_of_range", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 7\n")
    add("obj_face_zero_index", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n")
    add("obj_face_forward_reference", OBJ, b"v 0 0 0\nv 1 0 0\nf 1 2 3\nv 0 1 0\n")
    add("obj_face_negative_too_far", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf -1 -2 -4\n")
    add("obj_face_huge_index", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 99999999999999999999\n")
    add("obj_face_huge_negative", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 -99999999999999999999\n")
    add("obj_face_plus_sign", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf +1 +2 +3\n")
    add("obj_nul_in_index", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\x00junk\n")
    add("obj_repeated_vertex", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 2\n")
    add("obj_degenerate", OBJ, b"v 0 0 0\nv 1 0 0\nv 2 0 0\nf 1 2 3\n")
    add("obj_non_manifold", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nv 0 -1 0\nv 0 0 1\nf 1 2 3\nf 2 1 4\nf 1 2 5\n")
    add("obj_empty", OBJ, b"")
    add("obj_only_comments", OBJ, b"# nothing\n\n   \n")
    add("obj_vertices_only", OBJ, b"v 0 0 0\nv 1 0 0\n")
    add("obj_no_trailing_newline", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3")
    add("obj_first_error_wins", OBJ, b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 9\nv bad\nf 1 2\n")
    add("obj_vertical_tab_formfeed", OBJ, b"v\x0b0\x0c0 0\nv 1 0 0\nv 0 1 0\nf 1\x0b2\x0c3\n")
    P, F = grid(12, 9, jitter=0.1, seed=3)
    add("obj_grid12x9", OBJ, obj_text(P, F))
    add("obj_grid12x9_short_digits", OBJ, obj_text(P, F, "%.6g"))

    # ---- ASCII PLY (mesh_io.hpp:140-262, test_io.cpp:15-90)
    add("ply_ascii_square", PLY, PLY_ASCII_HEAD + SQUARE_PLY_BODY)
    add("ply_ascii_extra_props", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\nproperty float z\n"
        b"property uchar red\nelement face 1\nproperty list uchar int vertex_indices\nend_header\n"
        b"0 0 0 255\n1 0 0 0\n0 1 0 7\n3 0 1 2\n")
    add("ply_ascii_zyx_order_dup_x", PLY,
        b"ply\nformat ascii 1.0\ncomment c\nobj_info o\nelement vertex 3\nproperty float z\nproperty float y\n"
        b"property float x\nproperty float x\nelement face 1\nproperty list uchar int vertex_indices\nend_header\n"
        b"0 0 9 0\n0 0 9 1\n0 1 9 0\n3 0 1 2\n")
    add("ply_ascii_crlf", PLY, (PLY_ASCII_HEAD + SQUARE_PLY_BODY).replace(b"\n", b"\r\n"))
    add("ply_ascii_missing_magic", PLY, b"plo\n")
    add("ply_ascii_empty", PLY, b"")
    add("ply_ascii_no_end_header", PLY, b"ply\nformat ascii 1.0\nelement vertex 0\n")
    add("ply_ascii_quad", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 4\nproperty float x\nproperty float y\nproperty float z\n"
        b"element face 1\nproperty list uchar int vertex_indices\nend_header\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n4 0 1 2 3\n")
    add("ply_ascii_wrong_element_order", PLY,
        b"ply\nformat ascii 1.0\nelement face 0\nproperty list uchar int vertex_indices\n"
        b"element vertex 0\nproperty float x\nproperty float y\nproperty float z\nend_header\n")
    add("ply_ascii_big_endian", PLY, b"ply\nformat binary_big_endian 1.0\nend_header\n")
    add("ply_ascii_format_missing", PLY, b"ply\nformat\nend_header\n")
    add("ply_ascii_unknown_header_line", PLY, b"ply\nformat ascii 1.0\nbogus line here\n")
    add("ply_ascii_blank_header_line", PLY, b"ply\nformat ascii 1.0\n\nend_header\n")
    add("ply_ascii_property_before_element", PLY, b"ply\nformat ascii 1.0\nproperty float x\n")
    add("ply_ascii_bad_element", PLY, b"ply\nformat ascii 1.0\nelement vertex\n")
    add("ply_ascii_bad_element_count", PLY, b"ply\nformat ascii 1.0\nelement vertex four\n")
    add("ply_ascii_bad_list_property", PLY, b"ply\nformat ascii 1.0\nelement face 1\nproperty list uchar int\n")
    add("ply_ascii_bad_property", PLY, b"ply\nformat ascii 1.0\nelement vertex 1\nproperty float\n")
    add("ply_ascii_unsupported_type", PLY, b"ply\nformat ascii 1.0\nelement vertex 1\nproperty half x\n")
    add("ply_ascii_unsupported_list_type", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 1\nproperty list uchar long x\n")
    add("ply_ascii_negative_count", PLY,
        b"ply\nformat ascii 1.0\nelement vertex -1\nproperty float x\nproperty float y\nproperty float z\n"
        b"element face 0\nproperty list uchar int vertex_indices\nend_header\n")
    add("ply_ascii_missing_z", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\n"
        b"element face 0\nproperty list uchar int vertex_indices\nend_header\n0 0\n1 0\n0 1\n")
    add("ply_ascii_truncated_faces", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n1 1 0\n0 1 0\n3 0 1 2\n")
    add("ply_ascii_truncated_vertices", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n")
    add("ply_ascii_bad_scalar", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 q 0\n1 1 0\n0 1 0\n3 0 1 2\n3 0 2 3\n")
    add("ply_ascii_bad_list_count", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n1 1 0\n0 1 0\nx 0 1 2\n3 0 2 3\n")
    add("ply_ascii_bad_list_value", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n1 1 0\n0 1 0\n3 0 1\n3 0 2 3\n")
    add("ply_ascii_blank_record", PLY, PLY_ASCII_HEAD + b"0 0 0\n\n1 1 0\n0 1 0\n3 0 1 2\n3 0 2 3\n")
    add("ply_ascii_float_list_values", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n1 1 0\n0 1 0\n3.9 0 1 2.99\n3 0 2 3\n")
    add("ply_ascii_huge_list_count", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n1 1 0\n0 1 0\n1e300 0 1 2\n3 0 2 3\n")
    add("ply_ascii_negative_list_count", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n1 1 0\n0 1 0\n-2 0 1 2\n3 0 2 3\n")
    add("ply_ascii_index_out_of_range", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n1 1 0\n0 1 0\n3 0 1 2\n3 0 2 4\n")
    add("ply_ascii_negative_index", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n1 1 0\n0 1 0\n3 0 1 2\n3 0 -2 3\n")
    add("ply_ascii_trailing_lines", PLY, PLY_ASCII_HEAD + SQUARE_PLY_BODY + b"garbage line\n\n")
    add("ply_ascii_extra_tokens", PLY, PLY_ASCII_HEAD + b"0 0 0 9\n1 0 0 z\n1 1 0\n0 1 0\n3 0 1 2 7\n3 0 2 3\n")
    add("ply_ascii_extra_element", PLY,
        PLY_ASCII_HEAD.replace(b"end_header\n", b"element edge 2\nproperty int a\nproperty int b\nend_header\n")
        + SQUARE_PLY_BODY + b"0 1\n1 2\n")
    add("ply_ascii_extra_element_bad", PLY,
        PLY_ASCII_HEAD.replace(b"end_header\n", b"element edge 2\nproperty int a\nproperty int b\nend_header\n")
        + SQUARE_PLY_BODY + b"0 1\n1\n")
    add("ply_ascii_third_vertex_element", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\nproperty float z\n"
        b"element face 1\nproperty list uchar int vertex_indices\nelement vertex 1\nproperty float x\n"
        b"property float y\nproperty float z\nend_header\n0 0 0\n1 0 0\n1 1 0\n3 0 1 2\n0 1 0\n")
    add("ply_ascii_third_vertex_element_no_xyz", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\nproperty float z\n"
        b"element face 1\nproperty list uchar int vertex_indices\nelement vertex 1\nproperty float x\n"
        b"end_header\n0 0 0\n1 0 0\n1 1 0\n3 0 1 2\n0\n")
    add("ply_ascii_face_scalar_props", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\nproperty float z\n"
        b"element face 1\nproperty uchar flags\nproperty list uchar int vertex_indices\nproperty float q\n"
        b"end_header\n0 0 0\n1 0 0\n0 1 0\n7 3 0 1 2 0.5\n")
    add("ply_ascii_face_no_list", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\nproperty float z\n"
        b"element face 1\nproperty int a\nend_header\n0 0 0\n1 0 0\n0 1 0\n5\n")
    add("ply_ascii_two_face_lists", PLY,
        b"ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\nproperty float z\n"
        b"element face 1\nproperty list uchar int a\nproperty list uchar int b\nend_header\n"
        b"0 0 0\n1 0 0\n0 1 0\n2 0 1 3 0 1 2\n")
    add("ply_ascii_degenerate_face", PLY, PLY_ASCII_HEAD + b"0 0 0\n1 0 0\n2 0 0\n0 1 0\n3 0 1 2\n3 0 2 3\n")
    P, F = grid(10, 7, jitter=0.05, seed=5)
    add("ply_ascii_grid10x7", PLY, ply_ascii(P, F))

    # ---- binary PLY (device-decoded fixed layout + host walker paths)
    add("ply_bin_square", PLY, square_binary())
    add("ply_bin_square_crlf_header", PLY, square_binary().replace(b"\n", b"\r\n", 9))
    P, F = grid(16, 11, jitter=0.2, seed=7)
    vrows = [tuple(p) for p in P]
    frows = [([int(x) for x in f],) for f in F]
    add("ply_bin_grid16x11", PLY, ply_binary(_xyz_double(), vrows, _tri_list(), frows))
    add("ply_bin_grid_quality", PLY,
        ply_binary(_xyz_double() + [("double", "quality")], [tuple(p) + (float(i) * 0.5,) for i, p in enumerate(P)],
                   _tri_list(), frows))
    add("ply_bin_float32", PLY, ply_binary([("float", "x"), ("float", "y"), ("float", "z")], vrows, _tri_list(), frows))
    add("ply_bin_mixed_types", PLY,
        ply_binary([("uchar", "red"), ("float", "z"), ("short", "junk"), ("double", "x"), ("float64", "y")],
                   [(i % 256, p[2], -i, p[0], p[1]) for i, p in enumerate(P)],
                   [("uchar", "flags"), ("list", "ushort", "uint", "vertex_indices"), ("float", "q")],
                   [(1, [int(x) for x in f], 0.25) for f in F]))
    add("ply_bin_int_types", PLY,
        ply_binary([("int8", "x"), ("int16", "y"), ("uint", "z")], [(1, 0, 0), (0, 1, 0), (-3, -2, 7)],
                   [("list", "int", "short", "vertex_indices")], [([0, 1, 2],)]))
    add("ply_bin_uint8_indices", PLY, ply_binary(_xyz_double(), vrows[:3], _tri_list("uchar", "uchar"), [([0, 1, 2],)]))
    add("ply_bin_float_indices", PLY,
        ply_binary(_xyz_double(), vrows[:4], _tri_list("float", "double"), [([0.0, 1.9, 2.5],), ([0.0, 2.0, 3.99],)]))
    add("ply_bin_quad_face", PLY,
        ply_binary(_xyz_double(), vrows, _tri_list(), frows[:5] + [([0, 1, 2, 3],)] + frows[5:9]))
    add("ply_bin_two_vertex_face", PLY, ply_binary(_xyz_double(), vrows, _tri_list(), frows[:3] + [([0, 1],)] + frows[3:]))
    add("ply_bin_index_out_of_range", PLY,
        ply_binary(_xyz_double(), vrows, _tri_list(), frows[:7] + [([0, 1, len(vrows)],)] + frows[7:]))
    add("ply_bin_negative_index", PLY,
        ply_binary(_xyz_double(), vrows, _tri_list(), frows[:2] + [([0, -1, 2],)] + frows[2:]))
    add("ply_bin_nan_index", PLY,
        ply_binary(_xyz_double(), vrows[:3], _tri_list("uchar", "float"), [([0.0, float("nan"), 2.0],)]))
    add("ply_bin_nan_count", PLY,
        ply_binary(_xyz_double(), vrows[:3], _tri_list("float", "int"), [((float("nan"), [0, 1, 2]),)]))
    add("ply_bin_quad_then_range", PLY,
        ply_binary(_xyz_double(), vrows, _tri_list(), frows[:4] + [([0, 1, 999],), ([0, 1, 2, 3],)] + frows[4:]))
    full = ply_binary(_xyz_double(), vrows, _tri_list(), frows)
    head = full.index(b"end_header\n") + len(b"end_header\n")
    vbytes = 24 * len(vrows)
    add("ply_bin_truncated_in_vertices", PLY, full[:head + vbytes - 30])
    add("ply_bin_truncated_at_face_boundary", PLY, full[:head + vbytes + 13 * 20])
    add("ply_bin_truncated_mid_face", PLY, full[:head + vbytes + 13 * 20 + 6])
    add("ply_bin_truncated_no_faces", PLY, full[:head + vbytes])
    add("ply_bin_truncated_after_count", PLY, full[:head + vbytes + 13 * 3 + 1])
    quad_tail = ply_binary(_xyz_double(), vrows, _tri_list(), frows[:6] + [([0, 1, 2, 3, 4, 5, 6],)] + frows[6:8])
    cut = quad_tail.index(b"end_header\n") + 11 + vbytes + 13 * 6 + 1 + 4 * 5
    add("ply_bin_truncated_inside_long_list", PLY, quad_tail[:cut])
    add("ply_bin_bad_before_truncation", PLY,
        ply_binary(_xyz_double(), vrows, _tri_list(), frows[:3] + [([0, 1, 999],)] + frows[3:])[:head + vbytes + 13 * 9])
    add("ply_bin_trailing_garbage", PLY, full + b"\x01\x02garbage")
    add("ply_bin_test_io_truncated", PLY,
        b"ply\nformat binary_little_endian 1.0\nelement vertex 2\nproperty double x\nproperty double y\n"
        b"property double z\nelement face 0\nproperty list uchar int vertex_indices\nend_header\n" + b"\x00" * 24)
    add("ply_bin_no_vertices_no_faces", PLY, ply_binary(_xyz_double(), [], _tri_list(), []))
    add("ply_bin_vertices_no_faces", PLY, ply_binary(_xyz_double(), vrows[:5], _tri_list(), []))
    add("ply_bin_extra_element_lists", PLY,
        ply_binary(_xyz_double(), vrows, _tri_list(), frows,
                   extra_elements=[("material", [("list", "uchar", "float", "rgb"), ("int", "id")],
                                    [([0.5, 0.25], 1), ([1.0], 2)])]))
    add("ply_bin_extra_element_truncated", PLY,
        ply_binary(_xyz_double(), vrows, _tri_list(), frows,
                   extra_elements=[("material", [("list", "uchar", "float", "rgb"), ("int", "id")],
                                    [([0.5, 0.25], 1), ([1.0], 2)])])[:-3])
    add("ply_bin_vertex_list_after_xyz", PLY,
        ply_binary(_xyz_double() + [("list", "uchar", "int", "nbrs")], [tuple(p) + ([1, 2],) for p in vrows],
                   _tri_list(), frows))
    # (a list property BEFORE x/y/z makes the reference index its scalar list
    # out of bounds, mesh_io.hpp:244 -- undefined behaviour, rejected here,
    # so that layout is not part of the parity corpus)
    add("ply_bin_two_face_lists", PLY,
        ply_binary(_xyz_double(), vrows, [("list", "uchar", "int", "a"), ("list", "uchar", "int", "vertex_indices")],
                   [([9, 9], [int(x) for x in f]) for f in F]))
    add("ply_bin_third_face_element", PLY,
        ply_binary(_xyz_double(), vrows, _tri_list(), frows[:10],
                   extra_elements=[("face", _tri_list(), frows[10:20])]))
    add("ply_bin_no_xyz", PLY, ply_binary([("double", "x"), ("double", "y")], [(0.0, 0.0)], _tri_list(), []))
    add("ply_bin_face_no_list", PLY, ply_binary(_xyz_double(), vrows[:3], [("int", "a")], [(5,)]))
    add("ply_bin_repeated_vertex", PLY, ply_binary(_xyz_double(), vrows, _tri_list(), frows[:4] + [([5, 5, 6],)]))
    add("ply_bin_degenerate", PLY,
        ply_binary(_xyz_double(), [(0.0, 0, 0), (1.0, 0, 0), (2.0, 0, 0)], _tri_list(), [([0, 1, 2],)]))
    return C


def _mutate(rng: np.random.RandomState, data: bytes, alphabet: bytes, nmut: int) -> bytes:
    b = bytearray(data)
    for _ in range(nmut):
        op = rng.randint(4)
        pos = rng.randint(len(b) + 1) if b else 0
        ch = alphabet[rng.randint(len(alphabet))]
        if op == 0 and b:
            b[min(pos, len(b) - 1)] = ch
        elif op == 1:
            b.insert(pos, ch)
        elif op == 2 and b:
            del b[min(pos, len(b) - 1)]
        else:
            b = b[:pos]
    return bytes(b)


def fuzz_cases(seed: int = 1812060601, n_text: int = 160, n_bin: int = 120):
    """Seeded random mutations of small valid files (reference outcomes decide)."""
    rng = np.random.RandomState(seed)
    P, F = grid(3, 2, jitter=0.3, seed=11)
    bases_obj = [SQUARE_OBJ, obj_text(P, F, "%.9g"), b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf -3 -2 -1\n"]
    bases_ply = [PLY_ASCII_HEAD + SQUARE_PLY_BODY, ply_ascii(P, F)]
    text_alpha = b"0123456789 .-+eE/\n\r\t#vfxaply"
    out = []
    for i in range(n_text):
        if i % 2 == 0:
            base = bases_obj[rng.randint(len(bases_obj))]
            out.append(("fuzz_obj_%03d" % i, OBJ, _mutate(rng, base, text_alpha, 1 + rng.randint(3))))
        else:
            base = bases_ply[rng.randint(len(bases_ply))]
            out.append(("fuzz_ply_ascii_%03d" % i, PLY, _mutate(rng, base, text_alpha, 1 + rng.randint(3))))
    vrows = [tuple(p) for p in P]
    frows = [([int(x) for x in f],) for f in F]
    bases_bin = [ply_binary(_xyz_double(), vrows, _tri_list(), frows),
                 ply_binary([("float", "x"), ("float", "y"), ("float", "z")], vrows, _tri_list("uchar", "uint"), frows)]
    for i in range(n_bin):
        base = bases_bin[i % 2]
        head = base.index(b"end_header\n") + 11
        b = bytearray(base)
        op = rng.randint(3)
        if op == 0:  # flip bytes in the body
            for _ in range(1 + rng.randint(3)):
                j = head + rng.randint(len(b) - head)
                b[j] = rng.randint(256)
        elif op == 1:  # truncate the body
            b = b[:head + rng.randint(len(b) - head + 1)]
        else:  # set a face's count byte
            fstart = head + (24 if i % 2 == 0 else 12) * len(vrows)
            fs = 13
            k = rng.randint(len(frows))
            b[fstart + fs * k] = rng.choice([0, 1, 2, 3, 4, 255])
        out.append(("fuzz_ply_bin_%03d" % i, PLY, bytes(b)))
    return out


def all_cases():
    return hand_cases() + fuzz_cases()
