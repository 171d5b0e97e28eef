"""GAES v1 container round trip on a large record file: the reference CLI
(cmd_encrypt / cmd_decrypt in-process, compiled backend, all threads) vs the
reference CLI with the cuda backend registered vs this repo's vectorised
container path (paper_1506_08503_b200.container).  Same container bytes."""
import os
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [os.path.join(REPO, "baseline", "_ref"), REPO]
import gaes  # noqa: E402
from gaes import cli  # noqa: E402

from paper_1506_08503_b200 import container, plugin  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
rng = np.random.default_rng(7)
lens = rng.integers(1, 61, n)
alphabet = np.frombuffer(b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789 ", np.uint8)
body = alphabet[rng.integers(0, alphabet.size, int(lens.sum()))]
content = b"\n".join(body[o - l:o].tobytes() for o, l in zip(np.cumsum(lens), lens)) + b"\n"
key, iv = rng.bytes(16), rng.bytes(16)
tmp = tempfile.mkdtemp()
src, ctr, back = (os.path.join(tmp, x) for x in ("in.txt", "out.gaes", "back.txt"))
open(src, "wb").write(content)


def ref_cli():
    t0 = time.perf_counter()
    cli.main(["encrypt", "--key", key.hex(), "--iv", iv.hex(), "--in", src, "--out", ctr])
    t1 = time.perf_counter()
    cli.main(["decrypt", "--key", key.hex(), "--in", ctr, "--out", back])
    t2 = time.perf_counter()
    assert open(back, "rb").read() == content
    return t1 - t0, t2 - t1, open(ctr, "rb").read()


gaes.backend.select("compiled")
ref_cli()
enc_ref, dec_ref, blob_ref = ref_cli()
plugin.register(gaes_module=gaes, select=True)
ref_cli()  # first CUDA use in this process (context, tables, staging) outside the timing
enc_cc, dec_cc, blob_cc = ref_cli()
container.encrypt_records(content, key, iv=iv)  # warm
t0 = time.perf_counter()
blob = container.encrypt_records(content, key, iv=iv)
t1 = time.perf_counter()
plain = container.decrypt_container(blob, key)
t2 = time.perf_counter()
assert blob == blob_ref == blob_cc and plain == content
mb = len(content) / 1e6
print(f"{n} records, {mb:.1f} MB of record text, container {len(blob) / 1e6:.1f} MB (identical bytes)")
print(f"reference CLI, compiled backend : encrypt {enc_ref:.3f} s, decrypt {dec_ref:.3f} s")
print(f"reference CLI, cuda backend     : encrypt {enc_cc:.3f} s, decrypt {dec_cc:.3f} s")
print(f"container.py (this repo)        : encrypt {t1 - t0:.3f} s, decrypt {t2 - t1:.3f} s")
