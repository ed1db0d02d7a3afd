"""compute-sanitizer driver (SURVEY.md §4 layer 6, §5 race detection): one
small invocation of every stage of the path through the C ABI -- C1 and C2
single windows (FindRepeats), a 64-window C4 batch (batched FindRepeats, the
trace set, MATCH_ALL + REPLAY over the next ops) -- checked against the
oracle so a sanitizer run also proves the outputs unchanged.

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize.py [c1|c2|c4]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import oracle  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402


def check_window(ctx, S, min_len):
    rep, occ = ctx.find_repeats(torch.from_numpy(S).cuda(), min_len)
    ref = oracle.find_repeats(S, min_len, tier=1)["repeats"]
    got = [tuple(int(v) for v in r[:3]) for r in rep.cpu().numpy()]
    exp = [tuple(int(v) for v in r[:3]) for r in ref]
    assert got == exp, "repeats differ from the oracle"
    return len(got)


def main():
    which = sys.argv[1:] or ["c1", "c2", "c4"]
    ctx = Context(0)
    if "c1" in which:
        print("c1 repeats", check_window(ctx, gen.c1(), 5), flush=True)
    if "c2" in which:
        print("c2 repeats", check_window(ctx, gen.c2(), 25), flush=True)
    if "c4" in which:
        tok, off, st, so = gen.c4(windows=64)
        d, ds = torch.from_numpy(tok).cuda(), torch.from_numpy(st).cuda()
        rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
        roff_h = roff.cpu().numpy()
        for w in (0, 17, 63):
            ref = oracle.find_repeats(tok[off[w]:off[w + 1]], 25, tier=1)["repeats"]
            got = [tuple(int(v) for v in r[:3]) for r in rep[roff_h[w]:roff_h[w + 1]].cpu().numpy()]
            assert got == [tuple(int(v) for v in r[:3]) for r in ref], f"window {w} differs"
        trie = ctx.trie_build(d, off, rep, roff, 25, 0)
        hits = ctx.match(trie, ds, so, full=True)
        rp, nall = ctx.match(trie, ds, so, mode=1)
        assert nall == hits.shape[0]
        rp2 = ctx.replay(trie, hits, np.diff(so))
        assert torch.equal(rp, rp2), "apo_match mode 1 != apo_replay over the MATCH_ALL hits"
        print("c4(64) repeats", int(roff_h[-1]), "traces", trie.info()[0], "hits", nall, "replays", rp.shape[0],
              flush=True)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
