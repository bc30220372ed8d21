"""Model of fk_blur_tma's item / raw-buffer protocol (csrc/fk_blur_cols.cu): four warps walk the
blocks of a CTA's items; bytes of block k can be waited for once its request has been fired; the
buffer of block k is handed over -- the block nbuf ahead requested -- by warp k mod 4 once all four
warps have arrived at "H pass done"; the request cursor advances through the items using the
duty warp's own "next item" or the slot thread 0 published at the first block of the duty
warp's item; every warp picks up its next item from the previous item's slot at an item's first
block.  Random block counts (>= 2 per item) and random interleavings of the warps; checks that no
slot is read before it holds the item the reader wants, that the cursor is never more than two
items ahead of a hand-over, and that nobody waits forever.

Result: nbuf = 1 and 2 (what the kernel uses) hold with two slots; nbuf = 3 does not -- a warp
can then be a whole two-block item ahead of thread 0 and read a slot before thread 0 has
published it (the third raw buffer that was tried hung in the chunked host pipeline for this
reason); with every drawn item published three items ahead instead of two (`ahead` = 3, four
slots) three buffers hold as well -- measured: no faster, not kept.  usage: python tools/handover_model.py [cases]"""
import random
import sys


def run(nbuf, nitems, seed, nslots, ahead=2):
    rng = random.Random(seed)
    blocks = [rng.choice([2, 2, 2, 3, 4, 6]) for _ in range(nitems)]
    item_of, first = [], []
    for i, b in enumerate(blocks):
        first.append(len(item_of))
        item_of += [i] * b
    nblk = len(item_of)
    cur = dict(crb=0, citem=0, valid=nitems > 0)
    slots = [None] * nslots
    requested, handed = set(), set()
    pos = [(0, 0)] * 4          # per warp: (block, stage); stages: wait bytes, pick up / publish, H + arrive, duty, V
    arrived = [0] * nblk
    drawn = [ahead]             # thread 0 holds this item after the prologue
    if ahead == 3:
        slots[(0 - 1) % nslots] = 2   # the prologue publishes item 2 itself

    def request_next(item_no):
        if not cur["valid"]:
            return
        k = first[cur["citem"]] + cur["crb"]
        assert k not in requested and k < nblk
        requested.add(k)
        cur["crb"] += 1
        if cur["crb"] >= blocks[cur["citem"]]:
            cur["crb"] = 0
            cur["citem"] += 1
            rel = cur["citem"] - item_no
            assert rel in (1, 2), ("cursor lead", rel)
            if rel == 1:
                n = item_no + 1
            else:
                n = slots[(item_no + 2 - ahead) % nslots]
                assert n == item_no + 2, ("hand-over read slot", n, "wanted", item_no + 2)
            cur["valid"] = n < nitems

    for _ in range(nbuf):
        request_next(0)
    for _ in range(200000):
        runnable = []
        for w in range(4):
            k, st = pos[w]
            if k >= nblk:
                continue
            if st == 0 and k not in requested:
                continue
            if st == 3 and (k & 3) == w and arrived[k] < 4:
                continue
            runnable.append(w)
        if not runnable:
            return "ok" if all(p[0] >= nblk for p in pos) else ("deadlock", pos)
        w = rng.choice(runnable)
        k, st = pos[w]
        i = item_of[k]
        if st == 1 and k == first[i]:
            if i > 0:
                s = slots[(i + 1 - ahead) % nslots]
                assert s == i + 1, ("pick-up read slot", s, "wanted", i + 1)
            if w == 0:
                slots[i % nslots] = drawn[0]
                drawn[0] += 1
        elif st == 2:
            arrived[k] += 1
        elif st == 3 and (k & 3) == w:
            request_next(i)
            handed.add(k)
        pos[w] = (k + 1, 0) if st == 4 else (k, st + 1)
    return "no progress"


def check(nbuf, nslots, cases, ahead=2):
    bad = []
    for seed in range(cases):
        try:
            r = run(nbuf, random.Random(seed).randint(1, 12), seed, nslots, ahead)
        except AssertionError as e:
            r = e.args[0]
        if r != "ok":
            bad.append((seed, r))
    return bad


if __name__ == "__main__":
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    for nbuf, nslots, ahead in ((1, 2, 2), (2, 2, 2), (3, 4, 2), (3, 4, 3), (2, 4, 3), (1, 4, 3)):
        bad = check(nbuf, nslots, cases, ahead)
        print(f"nbuf {nbuf}, {nslots} slots, published {ahead} items ahead: {cases - len(bad)} of {cases} ok"
              + (f"; first failure {bad[0]}" if bad else ""))
