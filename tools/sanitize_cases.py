"""Small invocations of every kernel shape, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) on the GPU box:

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

Each case is checked against hashlib (tools/hostref.py) as well, so a clean sanitizer run
also confirms the results.  Inputs are sized so every batch sits exactly at
the end of its device allocation (no slack after the last message).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hostref  # noqa: E402  (hashlib checker)
from paper_2407_09333_b200 import _native, device  # noqa: E402

ALGS = ("sha1", "md5", "sm3")
ENV_KEYS = ("HB_TMA_CFG", "HB_SMALL_N", "HB_DIRECT_MAX_L", "HB_NO_SMALL_KERNEL", "HB_VARLEN_SORT", "HB_VARLEN_LD",
            "HB_VARLEN_BULK", "HB_VARLEN_PREFETCH", "HB_VC_STAGES", "HB_CHAIN_N", "HB_SORT_QMAJOR", "HB_VARLEN_PF",
            "HB_VARLEN_KERNEL", "HB_MD5_NB3_N", "HB_LATE_WAIT")


def with_env(env):
    for k in ENV_KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)
    _native.reload_tuning()  # the engine parses its knobs once; re-read them


def fixed(alg, n, L, flags=0):
    host = hostref.random_bytes(n * L, n + L).reshape(n, L)
    d = torch.from_numpy(host.copy()).cuda()
    got = device.hash_fixed(alg, d, flags=flags).cpu().numpy()
    assert np.array_equal(got, hostref.digests(alg, host)), (alg, n, L, flags)


def varlen(alg, n, maxlen, flags=0):
    lens = np.random.default_rng(n).integers(0, maxlen + 1, n).astype(np.int64)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    host = hostref.random_bytes(int(off[-1]), 7)
    d = torch.from_numpy(host.copy()).cuda()
    got = device.hash_varlen(alg, d, torch.from_numpy(off).cuda(), flags=flags, offset_base=0).cpu().numpy()
    assert np.array_equal(got, hostref.digests_varlen(alg, host, off)), (alg, n, maxlen, flags)


def main():
    cases = 0
    fixed_shapes = [({}, [(3000, 1024), (700, 1040), (300, 64), (300, 16), (300, 96), (257, 7), (129, 0)]),
                    ({"HB_CHAIN_N": "0"}, [(3000, 1024)]),
                    ({"HB_SMALL_N": "0", "HB_DIRECT_MAX_L": "0"}, [(5000, 64), (5000, 144)])]
    if _native.built_with_ab():
        fixed_shapes += [({"HB_TMA_CFG": "ws3x2"}, [(3000, 1024), (513, 80)]), ({"HB_TMA_CFG": "1x3"}, [(3000, 1024)])]
    for env, shapes in fixed_shapes:
        with_env(env)
        for alg in ALGS:
            for n, L in shapes:
                fixed(alg, n, L)
                cases += 1
    for alg in ALGS:
        fixed(alg, 2000, 1024, _native.HB_FLAG_NO_TMA)
        cases += 1
    # HB_FLAG_INPUT_READY: loads before griddepcontrol.wait, early release of
    # sub-wave grids; back-to-back flagged launches over independent inputs
    for alg in ALGS:
        for n, L in ((3000, 1024), (300, 64), (4099, 48), (1000, 256)):
            fixed(alg, n, L, _native.HB_FLAG_INPUT_READY)
            cases += 1
        ins = [torch.from_numpy(hostref.random_bytes(700 * 320, 90 + k).reshape(700, 320)).cuda() for k in range(4)]
        outs = [device.hash_fixed(alg, x, flags=_native.HB_FLAG_INPUT_READY) for x in ins]
        for x, o in zip(ins, outs):
            assert np.array_equal(o.cpu().numpy(), hostref.digests(alg, x.cpu().numpy()))
            cases += 1
    # MD5's single-warp two-messages-per-thread tile at any batch size, flagged
    # (early loads before griddepcontrol.wait) and unflagged
    for env in ({"HB_CHAIN_N": "0"}, {"HB_CHAIN_N": "0", "HB_MD5_NB3_N": "0"}, {"HB_LATE_WAIT": "0"}):
        with_env(env)
        for alg in ALGS:
            for n, L in ((3000, 1024), (700, 1040), (129, 144)):
                fixed(alg, n, L, _native.HB_FLAG_INPUT_READY)
                cases += 1
    varlen_arms = [({}, 0), ({"HB_VARLEN_SORT": "global"}, 0), ({"HB_VARLEN_SORT": "window"}, 0),
                   ({"HB_SORT_QMAJOR": "0"}, 0), ({"HB_VARLEN_PF": "0"}, 0)]
    if _native.built_with_ab():  # the A/B arms exist only in libhetoc_b200_ab.so
        varlen_arms += [({}, _native.HB_FLAG_VARLEN_COOP), ({}, _native.HB_FLAG_VARLEN_WORDS),
                        ({"HB_VARLEN_LD": "32"}, 0), ({"HB_VARLEN_BULK": "3"}, 0), ({"HB_VARLEN_PREFETCH": "1"}, 0),
                        ({"HB_VARLEN_KERNEL": "33"}, 0), ({"HB_VARLEN_KERNEL": "40"}, 0),
                        ({"HB_VARLEN_KERNEL": "47"}, 0), ({"HB_VARLEN_KERNEL": "49"}, 0),
                        ({"HB_VARLEN_KERNEL": "51"}, 0), ({"HB_VARLEN_KERNEL": "52"}, 0)]
    for env, fl in varlen_arms:
        with_env(env)
        for alg in ALGS:
            varlen(alg, 3000, 700, fl)
            varlen(alg, 40, 300, fl)
            cases += 2
    with_env({})
    # HB_FLAG_INPUT_READY varlen launches back to back on one scratch buffer:
    # MD5's sort overlaps the previous hash kernel's drain
    lens = np.random.default_rng(9).integers(0, 600, 3000).astype(np.int64)
    off = np.zeros(len(lens) + 1, np.int64)
    off[1:] = np.cumsum(lens)
    host = hostref.random_bytes(int(off[-1]), 11)
    d, d_off = torch.from_numpy(host.copy()).cuda(), torch.from_numpy(off).cuda()
    scratch = torch.empty(int(_native.lib().hb_varlen_scratch_bytes(len(lens))), dtype=torch.uint8, device="cuda:0")
    for alg in ALGS:
        outs = [device.hash_varlen(alg, d, d_off, scratch=scratch, flags=_native.HB_FLAG_INPUT_READY, offset_base=0)
                for _ in range(3)]
        ref = hostref.digests_varlen(alg, host, off)
        for o in outs:
            assert np.array_equal(o.cpu().numpy(), ref), alg
            cases += 1
    for alg in ALGS:
        for w in (9, 12):
            out = device.hash_decimal(alg, 5, 4000, w).cpu().numpy()
            assert np.array_equal(out, hostref.digests(alg, hostref.decimal_messages(5, 4000, w)))
            cases += 1
    # programmatic dependent launch: a chain of launches on one stream, each
    # consuming the previous one's digests, no host synchronisation between
    for L in (64, 1024):
        per = L // 32
        rows = per ** 3 if L > 64 else 1 << 10
        data = hostref.random_bytes(rows * L, 47).reshape(rows, L)
        cur, ref = torch.from_numpy(data).cuda(), data
        while rows >= per:
            rows //= per
            cur = device.hash_fixed("sm3", cur).reshape(rows, L)
            ref = hostref.digests("sm3", ref).reshape(rows, L)
            cases += 1
        assert np.array_equal(cur.cpu().numpy(), ref)
    # hb_digest_small: message in the launch parameters, digest + polled sequence word in mapped pinned memory
    from paper_2407_09333_b200.crypto import digest
    msg = hostref.random_bytes(4096, 53).tobytes()
    for alg in ALGS:
        for L in (0, 55, 56, 64, 256, 257, 4096):
            want = hostref.digests_varlen(alg, np.frombuffer(msg[:L], np.uint8), np.array([0, L], np.uint64))[0]
            assert digest(alg, msg[:L]).data == want.tobytes(), (alg, L)
            cases += 1
    # small untimed host calls: zero-copy reads of mapped pinned memory (hb_engine.cu small_batch)
    from paper_2407_09333_b200.crypto import batch_digest, batch_digest_varlen
    for alg in ALGS:
        for n, L in ((1, 64), (1000, 64), (64, 1024), (4096, 32), (33, 7)):
            rows = hostref.random_bytes(n * L, n * L).reshape(n, L)
            assert np.array_equal(batch_digest(alg, rows), hostref.digests(alg, rows)), (alg, n, L)
            cases += 1
        off = np.array([3, 3, 20, 21, 120, 4000], np.uint64)
        buf = hostref.random_bytes(4007, 3)
        assert np.array_equal(batch_digest_varlen(alg, buf, off), hostref.digests_varlen(alg, buf, off)), alg
        cases += 1
    torch.cuda.synchronize()
    print(f"sanitize cases ok: {cases} invocations bit-exact")


if __name__ == "__main__":
    main()
