"""Phase-accurate simulation of the attn_fwd mbarrier protocol (producer / MMA / 2 softmax
warpgroups) to find deadlocks before running on a GPU. MMAs complete instantly at issue
(commit arrives immediately); that is enough to expose ordering bugs."""
import random

KST, VST = 3, 2


class Bar:
    def __init__(self, count):
        self.count, self.pending, self.phase = count, count, 0

    def arrive(self):
        self.pending -= 1
        if self.pending == 0:
            self.phase += 1
            self.pending = self.count

    def done(self, parity):  # try_wait.parity: phase with parity `parity` has completed
        return (self.phase & 1) != parity


def cls_of(c, t):
    return (c >> (2 * t)) & 3


def run(units):
    B = dict(q_full=Bar(1), q_empty=Bar(1))
    for i in range(KST):
        B[f"k_full{i}"], B[f"k_empty{i}"] = Bar(1), Bar(1)
    for i in range(VST):
        B[f"v_full{i}"], B[f"v_empty{i}"] = Bar(1), Bar(1)
    for t in range(2):
        B[f"s_full{t}"], B[f"p_ready{t}"], B[f"o_full{t}"], B[f"o_empty{t}"] = Bar(1), Bar(1), Bar(1), Bar(1)

    def wait(name, parity):
        while not B[name].done(parity):
            yield name

    def producer():
        g = 0
        for it, steps in enumerate(units):
            yield from wait("q_empty", (it & 1) ^ 1)
            B["q_full"].arrive()
            for c in steps:
                ks, vs = g % KST, g % VST
                yield from wait(f"k_empty{ks}", ((g // KST) & 1) ^ 1)
                B[f"k_full{ks}"].arrive()
                yield from wait(f"v_empty{vs}", ((g // VST) & 1) ^ 1)
                B[f"v_full{vs}"].arrive()
                g += 1

    def mma():
        g = 0
        cnt_p, cnt_o = [0, 0], [0, 0]
        s_left = [0, 0]

        def issue_s(t, gs, li):
            B[f"s_full{t}"].arrive()
            s_left[li] -= 1
            if s_left[li] == 0:
                B[f"k_empty{gs % KST}"].arrive()
        for it, steps in enumerate(units):
            has = [any(cls_of(c, t) for c in steps) for t in range(2)]
            issued, first = [-1, -1], [True, True]
            yield from wait("q_full", it & 1)
            for j, c in enumerate(steps):
                vs = g % VST
                if issued[0] < j and issued[1] < j:
                    s_left[j & 1] = (1 if cls_of(c, 0) else 0) + (1 if cls_of(c, 1) else 0)
                if (cls_of(c, 0) and issued[0] < j) or (cls_of(c, 1) and issued[1] < j):
                    yield from wait(f"k_full{g % KST}", (g // KST) & 1)
                for t in range(2):
                    if cls_of(c, t) and issued[t] < j:
                        issue_s(t, g, j & 1)
                        issued[t] = j
                yield from wait(f"v_full{vs}", (g // VST) & 1)
                for t in range(2):
                    if not cls_of(c, t):
                        continue
                    yield from wait(f"p_ready{t}", cnt_p[t] & 1)
                    cnt_p[t] += 1
                    if first[t]:
                        yield from wait(f"o_empty{t}", (cnt_o[t] & 1) ^ 1)
                    first[t] = False
                    if j + 1 < len(steps) and cls_of(steps[j + 1], t):
                        g2 = g + 1
                        c2 = steps[j + 1]
                        if issued[0] <= j and issued[1] <= j:
                            s_left[(j + 1) & 1] = (1 if cls_of(c2, 0) else 0) + (1 if cls_of(c2, 1) else 0)
                        yield from wait(f"k_full{g2 % KST}", (g2 // KST) & 1)
                        issue_s(t, g2, (j + 1) & 1)
                        issued[t] = j + 1
                B[f"v_empty{vs}"].arrive()
                g += 1
            B["q_empty"].arrive()
            for t in range(2):
                if has[t]:
                    B[f"o_full{t}"].arrive()
                    cnt_o[t] += 1

    def softmax(t):
        cnt_s, cnt_o = 0, 0
        for steps in units:
            has = False
            for c in steps:
                if not cls_of(c, t):
                    continue
                yield from wait(f"s_full{t}", cnt_s & 1)
                cnt_s += 1
                B[f"p_ready{t}"].arrive()
                has = True
            if has:
                yield from wait(f"o_full{t}", cnt_o & 1)
                cnt_o += 1
                B[f"o_empty{t}"].arrive()

    roles = {"producer": producer(), "mma": mma(), "sm0": softmax(0), "sm1": softmax(1)}
    state = {k: None for k in roles}
    alive = set(roles)
    stuck = 0
    while alive:
        progressed = False
        for k in list(alive):
            try:
                w = next(roles[k])
                if w != state[k]:
                    progressed = True
                state[k] = w
            except StopIteration:
                alive.discard(k)
                progressed = True
        stuck = 0 if progressed else stuck + 1
        if stuck > 50:
            return {k: state[k] for k in alive}
    return None


if __name__ == "__main__":
    rng = random.Random(0)
    for trial in range(3000):
        units = []
        for _ in range(rng.randint(1, 4)):
            n = rng.randint(1, 9)
            steps = []
            for _ in range(n):
                c = 0
                while c == 0:
                    c = rng.choice([0, 1, 2]) | (rng.choice([0, 1, 2]) << 2)
                steps.append(c)
            units.append(steps)
        dl = run(units)
        if dl:
            print("DEADLOCK", units, dl)
            break
    else:
        print("no deadlock in 3000 random unit lists")
