"""Golden for a q_xi section whose alphabet exceeds 32.

compress() never writes codes >= 32, but a decoder reading foreign archives
must treat them as the reference does (codec.py:427-431: eq = tau' >>
min(code, K_MAX), 0 for code 31).  This script takes the reference's
archive of a golden field, rewrites some lossless vertices' code 31 as 40,
287 and 300 and some lossy codes as 33 (re-encoding q_xi with an alphabet
of 512), and records what the reference's decompress returns for it (or
its error).  Test infrastructure only.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
    NUMBA_CACHE_DIR=/tmp/vfcp_numba python oracle/gen_wide_codes_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
import vfcp  # noqa: E402  (the reference)
from vfcp import huffman  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def main():
    out = {}
    for tag, name in (("a", "cfg1_eps0.01"), ("b", "int3")):
        z = np.load(GOLDEN / f"field_{name}.npz")
        a = vfcp.Archive.from_bytes(z["archive"].tobytes())
        codes = huffman.decode(a.q_xi).astype(np.int64)
        ll31 = np.flatnonzero(codes == 31)
        codes[ll31[0::3]] = 40
        codes[ll31[1::3]] = 287
        codes[ll31[2::6]] = 300
        lossy = np.flatnonzero(codes < 31)
        codes[lossy[:5]] = 33      # eq = tau >> 30 = 0: l_d disagrees
        for variant, cd in (("ok", np.where(codes == 33, 0, codes)),
                            ("bad", codes)):
            b = vfcp.Archive(**{**a.__dict__,
                                "q_xi": huffman.encode(cd, 512)})
            blob = b.to_bytes()
            try:
                r = vfcp.reconstruct_fixed(vfcp.Archive.from_bytes(blob))
                recon = np.stack([r.u_fp, r.v_fp]).astype(np.int64)
                err = ""
            except ValueError as exc:
                recon = np.zeros((2, 0), np.int64)
                err = str(exc)
            out[f"{tag}_{variant}_archive"] = np.frombuffer(blob, np.uint8)
            out[f"{tag}_{variant}_recon"] = recon
            out[f"{tag}_{variant}_error"] = np.array(err)
            print(tag, variant, recon.shape, repr(err))
    np.savez_compressed(GOLDEN / "wide_codes.npz", **out)


if __name__ == "__main__":
    main()
