"""Product-side state layouts and synthetic keys (paper_2512_03644_b200/state.py)
pinned to the oracle: the keys are the reference's HashIn layouts
(evolution.cpp:21-31), the sizes its razor (ckpt.cpp:13-21,
evolution.cpp:15-19).  CPU only."""
import pyoracle as orc

from paper_2512_03644_b200 import state


def test_keys_match_the_oracle():
    for seed, dp, pp, tp in ((42, 0, 0, 0), (42, 7, 1, 3), (1, 65535, 2, 9)):
        assert state.optimizer_init(seed, dp, pp, tp, True) == orc.optimizer_init(seed, dp, pp, tp, True)
        assert state.optimizer_init(seed, dp, pp, tp, False) == orc.optimizer_init(seed, dp, pp, tp, False)
        assert state.weights_init(seed, pp, tp) == orc.weights_init(seed, pp, tp)
    # SURVEY 8(c) golden: optimizer_init(42, d0p0t0, true) = e515bfbd...60358c02
    assert state.optimizer_init(42, 0, 0, 0).hex().startswith("e515bfbd")
    assert state.optimizer_init(42, 0, 0, 0).hex().endswith("60358c02")


def test_zero3_llama3_8b_d8_layout():
    regs = state.zero3_shard(state.PHI_LLAMA3_8B, 8, dp=1)
    kinds = [r.kind for r in regs]
    assert kinds == [state.MASTER, state.ADAM_M, state.ADAM_V, state.PARAMS, state.CURSOR, state.RNG]
    adam = sum(r.nbytes for r in regs[:3])
    assert adam == orc.optimizer_bytes(state.PHI_LLAMA3_8B, 8, True) == 12_045_391_872
    assert regs[3].nbytes == 2_007_565_312
    assert state.shard_bytes(regs) == 14_052_957_184 + 32
    # distinct keys per region and per iteration
    keys = {r.digest for r in regs if r.digest} | {r.digest for r in state.zero3_shard(state.PHI_LLAMA3_8B, 8, 1,
                                                                                     iteration=2) if r.digest}
    assert len(keys) == 8


def test_zero3_ragged_division():
    # 12 phi / d not divisible: the three Adam regions still sum to ceil(12 phi / d)
    for phi, d in ((1001, 7), (5, 3), (123_457, 6)):
        regs = state.zero3_shard(phi, d, 0)
        assert sum(r.nbytes for r in regs[:3]) == orc.optimizer_bytes(phi, d, True)
        assert regs[3].nbytes == -(-2 * phi // d)


def test_region_specs_for_the_standby_tool():
    regs = state.zero3_shard(1 << 20, 2, 0)
    s = regs[0].spec().split(":")
    assert s[0] == str(state.MASTER) and int(s[1]) == regs[0].nbytes and len(s[2]) == 64
    c = regs[4].spec().split(":")
    assert c[2].startswith("=") and bytes.fromhex(c[2][1:]) == regs[4].literal
