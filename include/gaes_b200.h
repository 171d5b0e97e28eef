/*
 * gaes_b200.h -- C ABI of the B200-native AES-128 hot path (libgaes_b200.so).
 *
 * Drop-in boundary for the reference package `gaes` (arXiv 1506.08503,
 * /root/reference/pkg).  The reference's plug-in point is the backend
 * registry pkg/src/gaes/backend.py:17-64, whose modules export
 *     cbc_encrypt(data, ivs, round_keys, sbox, mix_lut, shift_src, out)
 *     cbc_decrypt(data, ivs, round_keys, inv_sbox, inv_mix_lut, inv_shift_src, out)
 * (pkg/src/gaes/_kernel.pyx:12-18 and :57-63).  gaes_cbc_encrypt /
 * gaes_cbc_decrypt below are exactly those two entry points flattened to
 * plain pointers and sizes; the ctypes module
 * paper_1506_08503_b200/backend_cuda.py binds them under NAME = "cuda".
 *
 * All functions return 0 on success or a negative GAES_E* code; the
 * message of the last failure on the calling thread is gaes_last_error().
 * Host-buffer entry points are synchronous (on return `out` is complete,
 * like the reference kernels); *_dev entry points are stream-ordered on
 * the cudaStream_t passed as `stream` (NULL = legacy default stream) and
 * take device pointers on the current device.
 *
 * Byte layout everywhere is the reference's (aes_cbc.py:3-5):
 * a 16-byte block is the AES state in FIPS-197 input order, byte 4c+r =
 * state row r, column c; round keys are u8[11][16] rows as returned by
 * key_schedule.KeySchedule.to_array() (key_schedule.py:35-38).
 */
#ifndef GAES_B200_H
#define GAES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GAES_API __attribute__((visibility("default")))

/* error codes */
#define GAES_OK 0
#define GAES_EINVAL -1   /* bad argument: mapped to ValueError            */
#define GAES_ECUDA -2    /* CUDA runtime failure: mapped to RuntimeError  */
#define GAES_ENODEV -3   /* no CUDA device visible: RuntimeError          */
#define GAES_ETABLE -4   /* GF-layer self check failed (sbox_gen.py:66-79) */

/* ---- library / device management ------------------------------------ */

/* ABI version (major*10000 + minor*100 + patch). */
GAES_API int gaes_version(void);
/* Message for the last failure on this thread ("" if none). */
GAES_API const char *gaes_last_error(void);
/* Number of visible CUDA devices (0 when none; never fails). */
GAES_API int gaes_device_count(void);
/* Number of GPUs the host-buffer entry points shard rows across
 * (contiguous balanced ranges, parallel.py:37-50 semantics).  n <= 0 or
 * n > device count selects all visible devices (the default).  With one
 * GPU the caller's current device is used (one process per GPU); with
 * several, devices 0 .. n-1.  Returns the number now in use. */
GAES_API int gaes_set_num_gpus(int n);
GAES_API int gaes_get_num_gpus(void);

/* ---- GF(2^8) layer (north_star (1); replaces sbox_gen.py:22-85 and
 *      aes_cbc.py:118-132,207-214 table construction) ------------------- */

/* Build S, S^-1 and the four-column T tables on `device` from field
 * arithmetic (gf256.py:38-75 multiply/inverse, sbox_gen.py affine maps,
 * circulant mix matrices (2,3,1,1)/(14,11,13,9)) and copy them to the host.
 * te[j*256+x] = pack_r M[r][j]*S[x]; td likewise with M^-1 and S^-1
 * (byte r of each little-endian word = state row r).  Any output pointer
 * may be NULL.  Returns GAES_ETABLE if the in-kernel cross checks (S^-1 o S
 * = id, M*M^-1 = I) fail. */
GAES_API int gaes_gf_tables(int device, uint8_t sbox[256], uint8_t inv_sbox[256],
                            uint32_t te[1024], uint32_t td[1024]);

/* 1 if (sbox, mix_lut, shift_src) equal the device GF layer's forward
 * tables, 0 if not, <0 on error.  Informational (the kernels accept any
 * tables; see gaes_cbc_encrypt). */
GAES_API int gaes_tables_are_standard(const uint8_t sbox[256], const uint8_t mix_lut[4096],
                                      const uint8_t shift_src[16], int decrypt);

/* The device GF layer's tables in the reference's backend-argument format
 * (what aes_cbc._encrypt_tables / _decrypt_tables hand to a backend,
 * aes_cbc.py:313-342): sbox u8[256] (S or S^-1), mix_lut u8[4][4][256]
 * (mix_lut[r][j][x] = M[r][j] * x for M = circ(2,3,1,1) or its inverse) and
 * shift_src u8[16].  Any pointer may be NULL. */
GAES_API int gaes_std_tables(int decrypt, uint8_t sbox[256], uint8_t mix_lut[4096], uint8_t shift_src[16]);

/* ---- reference backend contract (host buffers, synchronous) ----------
 * Replaces _kernel.cbc_encrypt (pkg/src/gaes/_kernel.pyx:12-54) and
 * _kernel_np.cbc_encrypt (_kernel_np.py:34-48).
 *   data, out : u8[n][m], C-contiguous, m % 16 == 0, m >= 16
 *   ivs       : u8[n][16] (per-row CBC start; a shared IV tiled by
 *               IVSet.rows is detected and folded into the round key)
 *   round_keys: u8[11][16] forward schedule (aes_cbc.py:333-342)
 *   sbox, mix_lut (u8[4][4][256], mix_lut[r][j][x] = m[r][j]*x),
 *   shift_src (u8[16], out[p] = in[shift_src[p]]) as handed over by
 *   aes_cbc._encrypt_tables.  Any tables are honoured: the T tables are
 *   built on the device from the ones passed.  n == 0 is a no-op.
 * Rows are sharded across gaes_get_num_gpus() devices.  Host buffers may
 * be pageable (staged through pinned ring buffers) or pinned (DMA direct).
 * Thread-safe; concurrent calls on disjoint rows are allowed
 * (parallel.py:66-75). */
GAES_API int gaes_cbc_encrypt(const uint8_t *data, const uint8_t *ivs, size_t n, size_t m,
                              const uint8_t round_keys[176], const uint8_t sbox[256],
                              const uint8_t mix_lut[4096], const uint8_t shift_src[16],
                              uint8_t *out);
/* Replaces _kernel.cbc_decrypt (_kernel.pyx:57-101); forward schedule,
 * inverse tables (aes_cbc.py:339-342). */
GAES_API int gaes_cbc_decrypt(const uint8_t *data, const uint8_t *ivs, size_t n, size_t m,
                              const uint8_t round_keys[176], const uint8_t inv_sbox[256],
                              const uint8_t inv_mix_lut[4096], const uint8_t inv_shift_src[16],
                              uint8_t *out);

/* Shared-IV form of the two calls above (IVSet.shared, aes_cbc.py:89-94)
 * using the device GF layer's standard tables: no N x 16 IV grid crosses
 * PCIe.  This is the end-to-end entry point bench.py times. */
GAES_API int gaes_encrypt_shared_iv(const uint8_t *data, size_t n, size_t m, const uint8_t iv[16],
                                    const uint8_t round_keys[176], uint8_t *out);
GAES_API int gaes_decrypt_shared_iv(const uint8_t *data, size_t n, size_t m, const uint8_t iv[16],
                                    const uint8_t round_keys[176], uint8_t *out);

/* Per-row IV form with the device GF layer's standard tables (no tables
 * crossing the boundary): ivs u8[n][16]; a shared IV tiled into rows is
 * detected and folded.  Used by the container path (per-message IVs,
 * container.py IV mode 0x01). */
GAES_API int gaes_cbc_encrypt_std(const uint8_t *data, const uint8_t *ivs, size_t n, size_t m,
                                  const uint8_t round_keys[176], uint8_t *out);
GAES_API int gaes_cbc_decrypt_std(const uint8_t *data, const uint8_t *ivs, size_t n, size_t m,
                                  const uint8_t round_keys[176], uint8_t *out);

/* Many-key batch with host buffers (config 5 end to end): key i owns rows
 * [i*blocks_per_key, (i+1)*blocks_per_key) of data/out (u8[k*bpk][16]);
 * keys u8[k][16] and per-key shared IVs u8[k][16] (NULL = zero IV) on the
 * host.  The key schedule runs on each GPU used (gaes_expand_keys_dev);
 * rows are sharded across gaes_get_num_gpus() devices. */
GAES_API int gaes_many_key_encrypt(const uint8_t *data, size_t blocks_per_key, size_t k, const uint8_t *keys,
                                   const uint8_t *ivs, uint8_t *out);
GAES_API int gaes_many_key_decrypt(const uint8_t *data, size_t blocks_per_key, size_t k, const uint8_t *keys,
                                   const uint8_t *ivs, uint8_t *out);

/* ---- device-resident entry points (stream-ordered, current device) ----
 * Standard tables from the device GF layer.  `iv` is a 16-byte HOST
 * array (shared IV, folded into the round keys) or NULL for a zero IV.
 * `out` may equal `in` or overlap it: where a kernel would read a block
 * another thread may already have overwritten (CBC decrypt of multi-block
 * rows in place, any partial overlap) the input is first copied to a
 * private stream-ordered buffer.  All of them are capturable into a CUDA
 * graph (no host synchronisation; captured launches read their input with
 * plain loads instead of a cached texture object). */

/* n_blocks independent 16-byte rows: out_i = E_K(in_i ^ iv)   (M = 16). */
GAES_API int gaes_encrypt_blocks_dev(const void *in, void *out, size_t n_blocks,
                                     const uint8_t round_keys[176], const uint8_t iv[16],
                                     void *stream);
/* out_i = D_K(in_i) ^ iv. */
GAES_API int gaes_decrypt_blocks_dev(const void *in, void *out, size_t n_blocks,
                                     const uint8_t round_keys[176], const uint8_t iv[16],
                                     void *stream);
/* General CBC over an n x m grid (m % 16 == 0).  ivs_dev: device u8[n][16]
 * per-row IVs, or NULL to use the shared host `iv` (NULL = zero IV).
 * Encrypt chains serially along each row; decrypt is block-parallel
 * (P_j = D(C_j) ^ C_{j-1}). */
GAES_API int gaes_cbc_encrypt_dev(const void *in, void *out, size_t n, size_t m,
                                  const void *ivs_dev, const uint8_t iv[16],
                                  const uint8_t round_keys[176], void *stream);
GAES_API int gaes_cbc_decrypt_dev(const void *in, void *out, size_t n, size_t m,
                                  const void *ivs_dev, const uint8_t iv[16],
                                  const uint8_t round_keys[176], void *stream);

/* ---- batched key schedule (north_star (3); replaces gen_keys,
 *      key_schedule.py:50-70, for K keys at once) -------------------- */

/* keys: device u8[k][16].  rk_enc: device u8[k][11][16], identical to
 * gen_keys(key_i, S).to_array().  rk_dec (nullable): device u8[k][11][16],
 * the equivalent-inverse-cipher form (rows 1..9 passed through
 * InvMixColumns; rows 0 and 10 unchanged). */
GAES_API int gaes_expand_keys_dev(const void *keys, size_t k, void *rk_enc, void *rk_dec,
                                  void *stream);

/* Many-key batch (config 5): key i owns blocks [i*bpk, (i+1)*bpk).
 * rk_enc / rk_dec as produced by gaes_expand_keys_dev; ivs_dev: device
 * u8[k][16] per-key shared IVs or NULL (zero IV). */
GAES_API int gaes_many_key_encrypt_dev(const void *in, void *out, size_t blocks_per_key, size_t k,
                                       const void *rk_enc, const void *ivs_dev, void *stream);
GAES_API int gaes_many_key_decrypt_dev(const void *in, void *out, size_t blocks_per_key, size_t k,
                                       const void *rk_dec, const void *ivs_dev, void *stream);

/* ---- measurement support ------------------------------------------------ */

/* Kernel launches issued by this library since load (bench "gpu_launches"). */
GAES_API uint64_t gaes_launch_count(void);
/* Name of the kernel variant the last M=16 encrypt used ("ttable_ilp2", ...). */
GAES_API const char *gaes_last_kernel(void);
/* Roofline probe: run the encrypt round function on register-resident
 * states (no HBM traffic), `iters` encryptions per thread on every SM, and
 * report the achieved table-lookup rate (160 lookups per encryption) -- the
 * measured ceiling of the shared-memory T-table formulation. */
GAES_API int gaes_probe_round_rate(int device, uint32_t iters, double *lookups_per_sec, double *ms);
/* Roofline denominator: the shared-memory lookup peak measured on this GPU
 * -- every lane of 1024-thread CTAs on all SMs streams conflict-free 4-byte
 * LDS (lane l hits bank l, as the table lookups do), `iters` x 16 per
 * thread; reports 4-byte lookups per second. */
GAES_API int gaes_probe_lds_peak(int device, uint32_t iters, double *lookups_per_sec, double *ms);
/* 1 if the standard-table kernels on `device` read round 10's S-box through
 * the texture path (144 shared-memory lookups + 16 texture fetches per
 * block), 0 if all 160 lookups are shared-memory (GAES_TUNE=TEXS=0), < 0 on
 * error.  Tells the roofline which lookups the L1/shared data pipe serves. */
GAES_API int gaes_uses_sbox_texture(int device);
/* Select the M=16 encrypt/decrypt formulation: 0 = auto (fastest measured),
 * 1 = T-table in shared memory, 2 = bitsliced.  Returns the value set or
 * GAES_EINVAL if the variant is not built. */
GAES_API int gaes_set_variant(int variant);
/* Host-runtime counters (tests / measurement; no reference counterpart).
 * Fills out[0..n) with, in order: copy pools created, parallel copy regions
 * run, most regions ever running at once, regions run on the caller's thread
 * because the pool was busy, texture objects created on the current device,
 * texture-cache entries on the current device, keys expanded by host
 * many-key jobs, shard runner threads (all devices).  Returns the number of
 * counters written. */
GAES_API int gaes_debug_counters(int64_t *out, int n);
/* Self-test of the host copy pool (no GPU needed): `regions` back-to-back
 * parallel regions of `parts` parts on a private pool of `workers` threads;
 * returns how many parts ran other than exactly once (0 = correct). */
GAES_API int64_t gaes_host_pool_selftest(int regions, int parts, int workers);

#ifdef __cplusplus
}
#endif
#endif /* GAES_B200_H */
