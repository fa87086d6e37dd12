"""CPU checks of bench.py's roofline cost model (no GPU): the constant-folded
ALU-op count of the paper's decimal workload against the per-block counts it
specialises."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_decimal_alu_ops_width9():
    assert [bench.alu_ops_decimal(a, 9) for a in ("md5", "sha1", "sm3")] == [127, 404, 1010]


def test_decimal_alu_ops_bounded_by_block_model():
    for alg in ("md5", "sha1", "sm3"):
        prev = 0
        for w in range(1, 56):
            ops = bench.alu_ops_decimal(alg, w)
            # more varying words never make the block cheaper; folding never
            # exceeds the arbitrary-data count (which adds 16 byte swaps for SHA-1/SM3)
            assert prev <= ops <= bench.ALU_OPS_PER_BLOCK[alg]
            prev = ops


def test_ncu_record_matches_the_kernel_that_ran():
    """roofline.traffic comes from the committed ncu record of the same kernel:
    ncu's demangled names and the library's are normalised alike, a workload
    reads its suite entry, and a record of another kernel is not used."""
    assert bench._kernel_key("void hb::k_varlen16l<1, false, -1, true>(unsigned char const*)") == \
        bench._kernel_key("void k_varlen16l<1, 0, (int)-1, 1>(const unsigned char *, const unsigned char *)")
    rec = bench.load_ncu("md5_1k")
    assert rec is not None and bench.load_ncu("md5_1k", rec["kernel"]) == rec
    assert bench.load_ncu("md5_1k", "void hb::k_generic<1, false>(unsigned char const*)") is None
    assert bench.load_ncu("varlen_md5")["kernel"] == bench.load_ncu("C4_varlen_md5")["kernel"]


def test_chain_bound_only_for_non_overlapping_steps():
    """The one-batch dependent-chain bound enters a fixed-width entry's
    roofline only when consecutive flagged steps cannot overlap on the GPU
    (long messages in a grid of fewer CTAs than SMs); varlen steps (the hash
    waits for its own sort) always keep it."""
    assert bench.pdl_overlap("fixed", 65536, 17)          # short messages: programmatic launches
    assert bench.pdl_overlap("fixed", 1 << 16, 1025)      # >= one CTA per SM
    assert not bench.pdl_overlap("fixed", 4096, 1025)     # sub-wave grid of long messages: plain launches
    assert not bench.pdl_overlap("varlen", 1 << 22, 65)
    assert not bench.pdl_overlap("decimal", 10 ** 9, 1)
