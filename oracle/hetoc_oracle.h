/*
 * hetoc_oracle.h -- CPU restatement of the reference hash path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 engine (paper_2407_09333_b200/csrc) and the CPU baseline arm of
 * bench.py.  The product path never links, loads or calls it; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may.  It is pinned against golden vectors produced by the reference
 * Python package itself (tests/golden/make_golden.py) and against the KATs in
 * SPEC.md:255-257.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference repo root).
 */
#ifndef HETOC_ORACLE_H
#define HETOC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_SHA1 = 0, ORC_MD5 = 1, ORC_SM3 = 2 };

/* DIGEST_LEN, pkg/src/hetoc/crypto/batch.py:23 */
int orc_digest_len(int alg);

/* Scalar single-message digests:
 *   sha1  pkg/src/hetoc/crypto/sha1.py:40-46
 *   md5   pkg/src/hetoc/crypto/md5.py:57-63
 *   sm3   pkg/src/hetoc/crypto/sm3.py:66-72                                   */
void orc_sha1(const uint8_t *msg, uint64_t len, uint8_t out[20]);
void orc_md5(const uint8_t *msg, uint64_t len, uint8_t out[16]);
void orc_sm3(const uint8_t *msg, uint64_t len, uint8_t out[32]);
/* digest(alg, message), pkg/src/hetoc/crypto/batch.py:102-109. -1 on bad alg. */
int orc_digest(int alg, const uint8_t *msg, uint64_t len, uint8_t *out);

/* batch_digest(alg, data), pkg/src/hetoc/crypto/batch.py:274-290: row i of the
 * fixed-width (n, msg_len) layout (batch.py:62, :77-83) -> out[i*dlen ..].
 * nthreads >= 1 splits [0,n) into np.linspace-style ranges (batch.py:305).   */
int orc_batch_fixed(int alg, const uint8_t *data, uint64_t n, uint64_t msg_len,
                    uint8_t *out, int nthreads);

/* Variable-length batch: message i = data[offsets[i], offsets[i+1]).  The
 * reference has no offsets layout; this is the per-message digest()
 * (batch.py:102-109) mapped over the offsets array.    */
int orc_batch_varlen(int alg, const uint8_t *data, const uint64_t *offsets,
                     uint64_t n, uint8_t *out, int nthreads);

/* Counter-based synthetic message bytes; identical to hb_fill_random_dev so
 * CPU tests can regenerate exactly what the GPU hashed.  byte_offset must be
 * a multiple of 8.                                                           */
void orc_fill_random(uint8_t *buf, uint64_t nbytes, uint64_t seed, uint64_t byte_offset);

/* gen_messages(start, count, width) bytes, pkg/src/hetoc/crypto/batch.py:86-99. */
int orc_gen_decimal(uint64_t start, uint64_t count, int width, uint8_t *out);

#ifdef __cplusplus
}
#endif
#endif
