"""Random structured mini-IR functions (the reference's textual IR,
SPEC.md:111-121) for fuzzing the GPU warp interpreter against the reference
interpreter: straight-line integer ops, divergent diamonds (nested), divergent
counted loops with phis, loads / stores with in- and out-of-bounds indices,
divisions that can fault, selects, and undef phi inputs.  SSA-valid by
construction (values leave a region only through phis).  Test helper."""
import random

BIN = ["add", "sub", "mul", "and", "or", "xor", "shl", "shr"]
CMP = ["icmp.eq", "icmp.ne", "icmp.lt", "icmp.gt", "icmp.le", "icmp.ge"]


class Gen:
    def __init__(self, seed):
        self.r = random.Random(seed)
        self.n = 0
        self.blocks = []          # (label, [lines])
        self.cur = None

    def val(self):
        self.n += 1
        return f"%v{self.n}"

    def label(self, tag):
        self.n += 1
        return f"{tag}{self.n}"

    def start(self, label):
        self.cur = (label, [])
        self.blocks.append(self.cur)

    def emit(self, line):
        self.cur[1].append("  " + line)

    def operand(self, scope):
        x = self.r.random()
        if x < 0.65 and scope:
            return self.r.choice(scope)
        return str(self.r.choice([0, 1, 2, 3, 5, 7, 16, 31, 33, 63, 64, -1, -7, 100000, -2147483648]))

    def straight(self, scope, count):
        for _ in range(count):
            k = self.r.random()
            v = self.val()
            if k < 0.45:
                self.emit(f"{v} = {self.r.choice(BIN)} {self.operand(scope)} {self.operand(scope)}")
            elif k < 0.55:
                self.emit(f"{v} = {self.r.choice(['div', 'rem'])} {self.operand(scope)} {self.operand(scope)}")
            elif k < 0.7:
                c = self.val()
                self.emit(f"{c} = {self.r.choice(CMP)} {self.operand(scope)} {self.operand(scope)}")
                self.emit(f"{v} = select {c} {self.operand(scope)} {self.operand(scope)}")
            elif k < 0.85:
                mem = self.r.choice(["ga", "gb", "sm"])
                idx = self.val()
                mask = self.r.choice(["63", "127", "31"])
                self.emit(f"{idx} = and {self.operand(scope)} {mask}")
                op = "load.shared" if mem == "sm" else "load.global"
                self.emit(f"{v} = {op} {mem} {idx}")
            else:
                mem = self.r.choice(["ga", "gb", "sm"])
                idx = self.val()
                self.emit(f"{idx} = and {self.operand(scope)} {self.r.choice(['63', '31', '15'])}")
                op = "store.shared" if mem == "sm" else "store.global"
                self.emit(f"{op} {mem} {idx} {self.operand(scope)}")
                continue
            scope.append(v)

    def region(self, scope, depth):
        """Emits a region starting in the current block; returns the new scope."""
        k = self.r.random()
        if depth >= 3 or k < 0.3:
            self.straight(scope, self.r.randint(1, 4))
            return scope
        if k < 0.75:                       # diamond
            c = self.val()
            self.emit(f"{c} = {self.r.choice(CMP)} {self.operand(scope)} {self.operand(scope)}")
            lt, lf, lj = self.label("t"), self.label("f"), self.label("j")
            self.emit(f"condbr {c} ^{lt} ^{lf}")
            outs = []
            for lab in (lt, lf):
                self.start(lab)
                sc = self.region(list(scope), depth + 1)
                self.straight(sc, self.r.randint(0, 2))
                outs.append((self.cur[0], sc[-1] if len(sc) > len(scope) else self.operand(scope)))
                self.emit(f"br ^{lj}")
            self.start(lj)
            v = self.val()
            a = outs[0][1] if self.r.random() > 0.1 else "undef"
            self.emit(f"{v} = phi {a}:^{outs[0][0]}, {outs[1][1]}:^{outs[1][0]}")
            return scope + [v]
        # counted loop with a lane-dependent trip count (divergent exit)
        pre = self.cur[0]
        lim = self.val()
        self.emit(f"{lim} = and {self.operand(scope)} 7")
        lh, lb, lx = self.label("h"), self.label("b"), self.label("x")
        self.emit(f"br ^{lh}")
        self.start(lh)
        i, acc, i1, acc1 = self.val(), self.val(), self.val(), self.val()
        a0 = self.operand(scope)
        body_end = [None]
        self.emit(f"{i} = phi 0:^{pre}, {i1}:^BODYEND")
        self.emit(f"{acc} = phi {a0}:^{pre}, {acc1}:^BODYEND")
        c = self.val()
        self.emit(f"{c} = icmp.lt {i} {lim}")
        self.emit(f"condbr {c} ^{lb} ^{lx}")
        self.start(lb)
        sc = self.region(list(scope) + [i, acc], depth + 1)
        self.emit(f"{acc1} = {self.r.choice(['add', 'xor', 'mul'])} {acc} {self.operand(sc)}")
        self.emit(f"{i1} = add {i} 1")
        self.emit(f"br ^{lh}")
        body_end[0] = self.cur[0]
        # patch the back-edge predecessor label
        hl = next(b for b in self.blocks if b[0] == lh)
        hl[1][:] = [ln.replace("BODYEND", body_end[0]) for ln in hl[1]]
        self.start(lx)
        return scope + [acc]

    def build(self):
        self.start("entry")
        self.emit("%t = tid")
        scope = ["%t", "%p"]
        for _ in range(self.r.randint(1, 4)):
            scope = self.region(scope, 0)
        ret = self.val()
        self.start(self.label("r")) if False else None
        self.emit(f"{ret} = add {self.operand(scope)} {self.operand(scope)}")
        self.emit(f"ret {ret}")
        body = "\n".join(f"^{lab}:\n" + "\n".join(lines) for lab, lines in self.blocks)
        return ("global ga[64]\nglobal gb[32]\n\nfn fuzz(%p) shared sm[48] {\n" + body + "\n}\n")


def random_function(seed):
    return Gen(seed).build()
