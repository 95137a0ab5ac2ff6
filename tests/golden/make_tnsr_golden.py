"""Generate tests/golden/tnsr_golden.json from the REAL reference's tensorfile
module (build container only; the GPU box uses the committed JSON).

Records, for the TNSR v1 format (/root/reference/pkg/src/rtcur/tensorfile.py):
* ``written``: the exact bytes the reference's ``write_tensor`` produces for a
  few seeded tensors (1..4 modes, special values);
* ``errors``: for malformed files (the reference test-suite's cases:
  bad magic/version, zero modes, zero extent, truncated header/extents/payload,
  trailing bytes, empty file, a video-scale header), the file bytes and the
  exact TensorFormatError text with the path replaced by ``{path}``;
* ``headers``: read_header results for the well-formed files.

Usage:  python tests/golden/make_tnsr_golden.py
"""

from __future__ import annotations

import json
import os
import struct
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_reference  # noqa: E402


def main():
    rtcur = _import_reference()
    from rtcur.tensor import DenseTensor
    from rtcur.tensorfile import TensorFormatError, read_header, read_tensor, write_tensor

    rng = np.random.default_rng(11)
    out = {"written": [], "errors": [], "headers": []}
    with tempfile.TemporaryDirectory() as tmp:
        cases = [((2, 3, 4), rng.standard_normal(24)), ((7,), rng.standard_normal(7)),
                 ((3, 5), rng.standard_normal(15)), ((2, 2, 2, 3), rng.standard_normal(24)),
                 ((6,), np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-308]))]
        for i, (shape, vals) in enumerate(cases):
            p = os.path.join(tmp, f"w{i}.tnsr")
            write_tensor(p, DenseTensor(vals, shape))
            raw = open(p, "rb").read()
            out["written"].append({"shape": list(shape), "hex": raw.hex()})
            v, dims = read_header(p)
            back = read_tensor(p)
            assert np.array_equal(back.data, np.asarray(vals, dtype=np.float64), equal_nan=True)
            out["headers"].append({"hex": raw.hex(), "version": v, "dims": list(dims)})

        def raw_file(dims, payload_count=None, version=1, magic=b"TNSR"):
            blob = magic + struct.pack("<HH", version, len(dims)) + struct.pack(f"<{len(dims)}Q", *dims)
            count = int(np.prod(dims)) if payload_count is None else payload_count
            return blob + np.arange(count, dtype="<f8").tobytes()

        bad = {
            "bad_magic": raw_file((2, 2), magic=b"XXXX"),
            "bad_magic_nonprint": raw_file((2, 2), magic=b"\x00T\xffS"),
            "bad_version": raw_file((2, 2), version=9),
            "zero_modes": b"TNSR" + struct.pack("<HH", 1, 0),
            "zero_extent": b"TNSR" + struct.pack("<HH", 1, 2) + struct.pack("<QQ", 3, 0),
            "truncated_header": b"TNSR" + struct.pack("<H", 1),
            "truncated_dims": b"TNSR" + struct.pack("<HH", 1, 3) + struct.pack("<Q", 4),
            "truncated_payload": raw_file((3, 4), payload_count=7),
            "trailing_bytes": raw_file((2, 2), payload_count=5),
            "video_scale": raw_file((256, 320, 3, 1250), payload_count=2),
            "one_mode_short": raw_file((5,), payload_count=4),
            "empty": b"",
        }
        for name, blob in bad.items():
            p = os.path.join(tmp, f"{name}.tnsr")
            with open(p, "wb") as f:
                f.write(blob)
            try:
                read_tensor(p)
                msg = None
            except TensorFormatError as exc:
                msg = str(exc).replace(p, "{path}")
            out["errors"].append({"name": name, "hex": blob.hex(), "message": msg})
    with open(os.path.join(HERE, "tnsr_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "tnsr_golden.json"), len(out["written"]), "files,", len(out["errors"]), "errors")


if __name__ == "__main__":
    main()
