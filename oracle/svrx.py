"""Test infrastructure (checker only, never on the product path): the SVRX
checkpoint container restated in numpy from the reference's
save_checkpoint / load_checkpoint (proj/src/io.cpp:229-359). io.cpp itself is
not built here (it needs libpng), so this restatement is the byte-level
checker for svr_scene_save_svrx / svr_scene_load_svrx.

Layout: "SVRX" | u32 version 1 | u32 header length | header JSON |
u64 code[N] | u8 level[N] | u32 corner_index[N][8] | f32 density[P] |
f32 sh[N][3(d+1)^2] | u32 zlib crc32 of everything before it. The header is
nlohmann::ordered_json::dump() of voxel_count, pool_count, sh_degree,
bounds_center, bounds_size (io.cpp:251-258)."""
import zlib

import numpy as np


def json_double(v: float) -> str:
    """nlohmann's float serialisation: shortest round-trip digits, '.0' on
    integral values, exponent form outside [1e-4, 1e15)."""
    v = float(v)
    if v == 0.0:
        return "-0.0" if np.signbit(v) else "0.0"
    mant, exp = f"{abs(v):.17e}".split("e")
    for prec in range(1, 18):
        txt = f"{abs(v):.{prec - 1}e}"
        if float(txt) == abs(v):
            mant, exp = txt.split("e")
            break
    d = mant.replace(".", "").rstrip("0") or "0"
    k, n = len(d), int(exp) + 1
    sign = "-" if v < 0 else ""
    if k <= n <= 15:
        return sign + d + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + d[:n] + "." + d[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + d
    e = n - 1
    return sign + d[0] + ("." + d[1:] if k > 1 else "") + f"e{'-' if e < 0 else '+'}{abs(e):02d}"


def encode(arrays) -> bytes:
    a = arrays
    bc = [json_double(x) for x in a.bounds_center]
    header = (f'{{"voxel_count":{a.n_voxels},"pool_count":{a.n_pool},"sh_degree":{int(a.sh_degree)},'
              f'"bounds_center":[{bc[0]},{bc[1]},{bc[2]}],"bounds_size":{json_double(a.bounds_size)}}}')
    h = header.encode()
    body = b"".join([b"SVRX", np.uint32(1).tobytes(), np.uint32(len(h)).tobytes(), h,
                     np.ascontiguousarray(a.codes, np.uint64).tobytes(),
                     np.ascontiguousarray(a.levels, np.uint8).tobytes(),
                     np.ascontiguousarray(a.corner_index, np.uint32).tobytes(),
                     np.ascontiguousarray(a.density, np.float32).tobytes(),
                     np.ascontiguousarray(a.sh, np.float32).tobytes()])
    return body + np.uint32(zlib.crc32(body)).tobytes()
