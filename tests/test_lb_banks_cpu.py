"""The shared-memory layouts of csrc/fwht_cols_lb.cu (large-block left
transform) are bank-optimal for every strip geometry: the round-1 staging
reads, the exchange writes / reads and the code-staging writes need no more
wavefronts than their byte counts (tools/lb_banks.py models the kernel's
address functions, including the lb_swz split into per-thread and
compile-time parts)."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _mod():
    spec = importlib.util.spec_from_file_location("lb_banks", os.path.join(ROOT, "tools", "lb_banks.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_lb_layouts_bank_optimal():
    m = _mod()
    for es, LB, E in ((2, 9, 16384), (2, 10, 32768), (2, 11, 32768), (2, 12, 32768),
                      (4, 9, 16384), (4, 10, 16384), (4, 11, 16384), (4, 12, 16384)):
        bad, _ = m.run(LB, E, es)
        assert max(bad.values()) == 0, (es, LB, bad)


def test_lb_swizzle_split_identity():
    """lb_swz(64a + b, cp) == lb_hi(a) ^ lb_lo(b, cp) (the kernel's hot-loop form)."""
    def swz(r, cp, RB, INL):
        f = (((r >> 6) << (0 if RB == 16 else 1)) ^ (r >> INL)) & 7
        return (r * RB + 8 * cp) ^ (f << 4)

    def hi(a, RB):
        return (64 * RB * a) ^ ((((a << (0 if RB == 16 else 1)) & 7)) << 4)

    def lo(b, cp, RB, INL):
        return (b * RB + 8 * cp) ^ (((b >> INL) & 7) << 4)
    for RB, INL in ((16, 3), (32, 2), (64, 1), (128, 0), (256, 0)):
        for a in range(0, 64, 3):
            for b in range(64):
                for cp in range(RB // 8):
                    assert swz(64 * a + b, cp, RB, INL) == hi(a, RB) ^ lo(b, cp, RB, INL)
