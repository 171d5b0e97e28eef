"""Generate tests/golden/ fixtures by running the REFERENCE package itself.

Run here (the container with /root/reference mounted), never on the GPU box:

    python tests/golden/make_golden.py

It imports the reference ``gaes`` package -- from ``baseline/_ref`` (the
pip-installed, compiled reference) if present, else straight from
/root/reference/pkg/src with its numpy backend -- and records:

* the cipher tables the reference hands to its backend
  (aes_cbc.py:316-342: sbox, inv_sbox, mix LUTs, shift permutations);
* round keys from key_schedule.gen_keys for the FIPS-197 key, the zero key
  and 256 seeded random keys (test_key_schedule.py:28-54 style);
* CBC cases through the reference's public entry points
  (aes_cbc.encrypt_batch / decrypt_batch): ragged (n, blocks) grids with
  shared and per-message IVs, mirroring test_backends.py:21-42 and
  test_aes_cbc.py:258-296;
* digests of the north-star configs at seed 2016 (bench.py:124-126 recipe):
  N = 2**16 in full, and N = 2**24 (digest only).

Outputs: tests/golden/golden.npz and tests/golden/golden.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def _import_reference():
    ref_installed = os.path.join(REPO, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_installed, "gaes")):
        sys.path.insert(0, ref_installed)
    else:
        sys.path.insert(0, "/root/reference/pkg/src")
    import gaes  # noqa: F401
    from gaes import aes_cbc, backend, key_schedule, sbox_gen
    return gaes, aes_cbc, backend, key_schedule, sbox_gen


def main():
    gaes, aes_cbc, backend, key_schedule, sbox_gen = _import_reference()
    print("reference backend:", backend.name(), "from", os.path.dirname(gaes.__file__))
    shared = aes_cbc._shared_arrays()
    fx = {
        "sbox": np.array(shared["forward"]),
        "inv_sbox": np.array(shared["inverse"]),
        "mix_fwd": np.array(shared["mix_fwd"]),
        "mix_inv": np.array(shared["mix_inv"]),
        "shift": np.array(shared["shift"]),
        "inv_shift": np.array(shared["inv_shift"]),
        "rcon": np.frombuffer(key_schedule.round_constants(), np.uint8).copy(),
    }
    fwd = sbox_gen.default_pair().forward

    rng = np.random.default_rng(1506)
    keys = [bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c"), bytes(16),
            bytes.fromhex("000102030405060708090a0b0c0d0e0f")]
    keys += [rng.bytes(16) for _ in range(253)]
    fx["keys"] = np.frombuffer(b"".join(keys), np.uint8).reshape(-1, 16).copy()
    fx["round_keys"] = np.stack([key_schedule.gen_keys(k, fwd).to_array() for k in keys])

    # CBC cases through the public entry points.
    cases = [(1, 1), (3, 1), (1, 5), (17, 3), (64, 2), (5, 4), (32, 2), (257, 1),
             (1000, 1), (31, 7), (2, 16)]
    meta = []
    for idx, (n, blocks) in enumerate(cases):
        crng = np.random.default_rng(9000 + idx)
        key = crng.bytes(16)
        data = crng.integers(0, 256, (n, 16 * blocks), dtype=np.uint8)
        per_msg = idx % 2 == 1
        if per_msg:
            ivrows = crng.integers(0, 256, (n, 16), dtype=np.uint8)
            ivs = aes_cbc.IVSet.per_message(ivrows)
        else:
            iv = crng.bytes(16)
            ivs = aes_cbc.IVSet.shared(iv)
            ivrows = ivs.rows(n)
        batch = aes_cbc.MessageBatch(data=data, original_lens=(16 * blocks,) * n)
        ct = aes_cbc.encrypt_batch(key, ivs, batch)
        pt = aes_cbc.decrypt_batch(key, ivs, ct)
        assert np.array_equal(pt, data)
        fx[f"case{idx}_key"] = np.frombuffer(key, np.uint8).copy()
        fx[f"case{idx}_pt"] = data
        fx[f"case{idx}_iv"] = np.ascontiguousarray(ivrows)
        fx[f"case{idx}_ct"] = ct
        meta.append({"idx": idx, "n": n, "blocks": blocks, "iv": "per-message" if per_msg else "shared"})

    # north-star config digests (seed 2016, bench.py:124-126 draw order)
    digests = {}
    for log_n in (16, 24):
        n = 1 << log_n
        drng = np.random.default_rng(2016)
        key = drng.bytes(16)
        iv = drng.bytes(16)
        p = drng.integers(0, 256, (n, 16), dtype=np.uint8)
        tables = aes_cbc._encrypt_tables(key)
        ivrows = aes_cbc.IVSet.shared(iv).rows(n)
        out = np.empty_like(p)
        backend.cbc_encrypt(p, ivrows, *tables, out)
        digests[str(n)] = {
            "seed": 2016, "key": key.hex(), "iv": iv.hex(),
            "sha256_p": hashlib.sha256(p.tobytes()).hexdigest(),
            "sha256_c": hashlib.sha256(out.tobytes()).hexdigest(),
            "c_first": out[0].tobytes().hex(), "c_last": out[-1].tobytes().hex(),
        }
        if log_n == 16:
            fx["cfg1_ct_rows_0_64"] = out[:64].copy()
        print(n, digests[str(n)]["sha256_c"])

    # GAES v1 containers (container.py / cli.py paths), test_container.py recipe
    from gaes import cli, container
    gkey = bytes.fromhex("000102030405060708090a0b0c0d0e0f")
    giv = bytes.fromhex("f0e1d2c3b4a5968778695a4b3c2d1e0f")
    gmsgs = [b"alpha", b"bravo-bravo", b"charlie charlie charlie!"]
    gb = aes_cbc.pad_zero(gmsgs)
    gsiv = aes_cbc.IVSet.shared(giv)
    blob = container.container_bytes(container.CipherContainer(
        iv_set=gsiv, original_lens=gb.original_lens, payload=aes_cbc.encrypt_batch(gkey, gsiv, gb)))
    fx["container_golden"] = np.frombuffer(blob, np.uint8).copy()
    # a records file: newline-separated records of varied lengths
    rrng = np.random.default_rng(4242)
    recs = []
    for _ in range(300):
        ln = int(rrng.integers(1, 70))
        r = rrng.integers(0, 256, ln, dtype=np.uint8)
        r[r == 0x0A] = 0x0B
        recs.append(r.tobytes())
    content = b"\n".join(recs) + b"\n"
    rkey, riv = rrng.bytes(16), rrng.bytes(16)
    records = cli._split_records(content)
    rb = aes_cbc.pad_zero(records)
    rsiv = aes_cbc.IVSet.shared(riv)
    shared_blob = container.container_bytes(container.CipherContainer(
        iv_set=rsiv, original_lens=rb.original_lens, payload=aes_cbc.encrypt_batch(rkey, rsiv, rb)))
    pivs = rrng.integers(0, 256, (rb.n_messages, 16), dtype=np.uint8)
    rpiv = aes_cbc.IVSet.per_message(pivs)
    per_blob = container.container_bytes(container.CipherContainer(
        iv_set=rpiv, original_lens=rb.original_lens, payload=aes_cbc.encrypt_batch(rkey, rpiv, rb)))
    fx["records_content"] = np.frombuffer(content, np.uint8).copy()
    fx["records_key"] = np.frombuffer(rkey, np.uint8).copy()
    fx["records_iv"] = np.frombuffer(riv, np.uint8).copy()
    fx["records_ivs"] = pivs
    fx["records_shared_container"] = np.frombuffer(shared_blob, np.uint8).copy()
    fx["records_permsg_container"] = np.frombuffer(per_blob, np.uint8).copy()
    digests["container_golden_sha256"] = hashlib.sha256(blob).hexdigest()

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **fx)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference_backend": backend.name(),
                   "cases": meta, "digests": digests}, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
