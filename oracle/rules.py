"""Exact bilinear rules <U,V,W> and their analysis -- ORACLE side.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares nothing with the CUDA product path.

Conventions (Eq. eqn:bilinear_alg and the sentence after it): a rule
<M0,K0,N0;R> is given by U (M0K0 x R), V (K0N0 x R), W (M0N0 x R) with
  * U rows = entries of A in COLUMN-major order:  i = ia + M0*ja
  * V rows = entries of B in COLUMN-major order:  j = ja + K0*jb
  * W rows = entries of C in ROW-major order:     k = ia*N0 + jb
Coefficients are exact Fractions.

Everything here is plain Python on tiny integer/rational tables.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from itertools import product
from typing import Sequence

import numpy as np


@dataclass(frozen=True)
class Rule:
    name: str
    m0: int
    k0: int
    n0: int
    U: tuple  # tuple of tuples of Fraction, shape (m0*k0, R)
    V: tuple  # (k0*n0, R)
    W: tuple  # (m0*n0, R)

    @property
    def R(self) -> int:
        return len(self.U[0])

    def as_float(self):
        """U, V, W as float64 numpy arrays (exact for dyadic coefficients)."""
        f = lambda X: np.array([[float(x) for x in row] for row in X], dtype=np.float64)
        return f(self.U), f(self.V), f(self.W)


def _frac_rows(rows) -> tuple:
    return tuple(tuple(Fraction(x) for x in r) for r in rows)


def make_rule(name, m0, k0, n0, U, V, W) -> Rule:
    U, V, W = _frac_rows(U), _frac_rows(V), _frac_rows(W)
    R = len(U[0])
    assert len(U) == m0 * k0 and len(V) == k0 * n0 and len(W) == m0 * n0, name
    assert all(len(r) == R for r in U + V + W), name
    return Rule(name, m0, k0, n0, U, V, W)


# ---------------------------------------------------------------------------------------------
# Built-in rules
# ---------------------------------------------------------------------------------------------

def classical222() -> Rule:
    """Classical <2,2,2;8>: product r = 4*ia + 2*ja + jb is A(ia,ja)*B(ja,jb) into C(ia,jb)
    (the rule whose recursion is the classical algorithm; Table 1 row 'classical')."""
    R = 8
    U = [[0] * R for _ in range(4)]
    V = [[0] * R for _ in range(4)]
    W = [[0] * R for _ in range(4)]
    for ia, ja, jb in product(range(2), repeat=3):
        r = 4 * ia + 2 * ja + jb
        U[ia + 2 * ja][r] = 1
        V[ja + 2 * jb][r] = 1
        W[ia * 2 + jb][r] = 1
    return make_rule("classical222", 2, 2, 2, U, V, W)


# Appendix A as PRINTED.  Its rows are A11,A12,A21,A22 for U/V and
# C11,C21,C12,C22 for W -- the transposed convention (reading A1).
STRASSEN_APP_A_PRINTED = (
    [[1, 0, 1, 0, 1, -1, 0],
     [0, 0, 0, 0, 1, 0, 1],
     [0, 1, 0, 0, 0, 1, 0],
     [1, 1, 0, 1, 0, 0, -1]],
    [[1, 1, 0, -1, 0, 1, 0],
     [0, 0, 1, 0, 0, 1, 0],
     [0, 0, 0, 1, 0, 0, 1],
     [1, 0, -1, 0, 1, 0, 1]],
    [[1, 0, 0, 1, -1, 0, 1],
     [0, 1, 0, 1, 0, 0, 0],
     [0, 0, 1, 0, 1, 0, 0],
     [1, -1, 1, 0, 0, 1, 0]],
)


def _swap_rows_1_2(X):
    X = [list(r) for r in X]
    X[1], X[2] = X[2], X[1]
    return X


def strassen() -> Rule:
    """Strassen <2,2,2;7> from App. A converted to the stated convention
    by swapping rows 2 and 3 (1-based) of U, V and W, i.e. the vec-permutation P_{2,2}
    (reading A1).  Products in the paper's numbering:
    M1=(A11+A22)(B11+B22), M2=(A21+A22)B11, M3=A11(B12-B22), M4=A22(B21-B11),
    M5=(A11+A12)B22, M6=(A21-A11)(B11+B12), M7=(A12-A22)(B21+B22)."""
    U, V, W = (_swap_rows_1_2(X) for X in STRASSEN_APP_A_PRINTED)
    return make_rule("strassen", 2, 2, 2, U, V, W)


def winograd() -> Rule:
    """Strassen-Winograd <2,2,2;7> (named at P:76; coefficients not printed
    in the paper -- DESIGN.md reading A2).  Written from its products:
      M1=A11 B11, M2=A12 B21, M3=(A11-A21+A12-A22) B22, M4=A22 (B11-B21-B12+B22),
      M5=(A21+A22)(B12-B11), M6=(A21+A22-A11)(B11-B12+B22), M7=(A11-A21)(B22-B12);
      C11=M1+M2, C12=M1+M3+M5+M6, C21=M1-M4+M6+M7, C22=M1+M5+M6+M7.
    Pinned by the Brent equations (tests), not by a printed table."""
    # rows: U (A11, A21, A12, A22); V (B11, B21, B12, B22); W (C11, C12, C21, C22)
    U = [[1, 0, 1, 0, 0, -1, 1],
         [0, 0, -1, 0, 1, 1, -1],
         [0, 1, 1, 0, 0, 0, 0],
         [0, 0, -1, 1, 1, 1, 0]]
    V = [[1, 0, 0, 1, -1, 1, 0],
         [0, 1, 0, -1, 0, 0, 0],
         [0, 0, 0, -1, 1, -1, -1],
         [0, 0, 1, 1, 0, 1, 1]]
    W = [[1, 1, 0, 0, 0, 0, 0],
         [1, 0, 1, 0, 1, 1, 0],
         [1, 0, 0, -1, 0, 1, 1],
         [1, 0, 0, 0, 1, 1, 1]]
    return make_rule("winograd", 2, 2, 2, U, V, W)


def _kron_rows(P: np.ndarray, Q: np.ndarray, X) -> list:
    """(P (x) Q) X for integer/Fraction tables X (rows permuted/combined)."""
    K = np.kron(P, Q).astype(int)
    Xa = np.array([[Fraction(x) for x in r] for r in X], dtype=object)
    return (K.astype(object) @ Xa).tolist()


SWAP2 = np.array([[0, 1], [1, 0]])
I2 = np.eye(2, dtype=int)


def strassen_dalberto() -> Rule:
    """D'Alberto's variant: <U, (swap (x) I2) V, (I2 (x) swap) W> of Strassen."""
    s = strassen()
    V = _kron_rows(SWAP2, I2, s.V)
    W = _kron_rows(I2, SWAP2, s.W)
    return make_rule("strassen_dalberto", 2, 2, 2, s.U, V, W)


def castrapel_gustafson(base: Rule, x: int, y: int, z: int) -> Rule:
    """Castrapel-Gustafson variants: <(P^x (x) P^y) U, (P^z (x) P^x) V,
    (P^y (x) P^z) W> with P = swap, x, y, z in {1, 2}."""
    p = lambda e: np.linalg.matrix_power(SWAP2, e).astype(int)
    U = _kron_rows(p(x), p(y), base.U)
    V = _kron_rows(p(z), p(x), base.V)
    W = _kron_rows(p(y), p(z), base.W)
    return make_rule(f"{base.name}_cg{x}{y}{z}", base.m0, base.k0, base.n0, U, V, W)


def make_rule_labelled(name, m0, k0, n0, U, V, W, u_labels, v_labels, w_labels,
                       u_den=1, v_den=1, w_den=1) -> Rule:
    """A rule from tables whose rows are given in an arbitrary order: row p of U is the entry
    u_labels[p] = (ia, ja) of A, row p of V is v_labels[p] = (ja, jb) of B, row p of W is
    w_labels[p] = (ia, jb) of C; entries are divided by the *_den prefactors.  Rows are placed
    in the stated convention: U row ia + m0*ja, V row ja + k0*jb, W row ia*n0 + jb.
    Used for App. C's <4,4,2;26>, whose printed row order is not that
    convention (reading A27)."""
    R = len(U[0])

    def place(X, labels, nrows, index, den):
        out = [None] * nrows
        for row, lab in zip(X, labels):
            out[index(*lab)] = [Fraction(x, den) for x in row]
        assert all(r is not None for r in out) and len(labels) == nrows, name
        return out

    Uo = place(U, u_labels, m0 * k0, lambda ia, ja: ia + m0 * ja, u_den)
    Vo = place(V, v_labels, k0 * n0, lambda ja, jb: ja + k0 * jb, v_den)
    Wo = place(W, w_labels, m0 * n0, lambda ia, jb: ia * n0 + jb, w_den)
    assert all(len(r) == R for r in Uo + Vo + Wo)
    return make_rule(name, m0, k0, n0, Uo, Vo, Wo)


BUILTINS = {
    "classical222": classical222,
    "strassen": strassen,
    "winograd": winograd,
    "strassen_dalberto": strassen_dalberto,
}


def builtin(name: str) -> Rule:
    return BUILTINS[name]()


# ---------------------------------------------------------------------------------------------
# Brent equations (exact): sum_r U_ir V_jr W_kr = 1 iff A-entry i, B-entry j, C-entry k form a
# classical product term a(ia,ja) b(ja,jb) -> c(ia,jb), else 0 (correctness of
# Eq. eqn:bilinear_alg for all A, B).
# ---------------------------------------------------------------------------------------------

def brent_violations(rule: Rule, conv=("col", "col", "row")) -> list:
    """List of violated (i, j, k) triples under the given row conventions for (U, V, W)."""
    m0, k0, n0, R = rule.m0, rule.k0, rule.n0, rule.R

    def a_idx(i):  # -> (ia, ja)
        return (i % m0, i // m0) if conv[0] == "col" else (i // k0, i % k0)

    def b_idx(j):  # -> (ja, jb)
        return (j % k0, j // k0) if conv[1] == "col" else (j // n0, j % n0)

    def c_idx(k):  # -> (ia, jb)
        return (k // n0, k % n0) if conv[2] == "row" else (k % m0, k // m0)

    bad = []
    for i in range(m0 * k0):
        ia, ja = a_idx(i)
        for j in range(k0 * n0):
            ja2, jb = b_idx(j)
            for k in range(m0 * n0):
                ia2, jb2 = c_idx(k)
                s = sum(rule.U[i][r] * rule.V[j][r] * rule.W[k][r] for r in range(R))
                want = 1 if (ja == ja2 and ia == ia2 and jb == jb2) else 0
                if s != want:
                    bad.append((i, j, k))
    return bad


# ---------------------------------------------------------------------------------------------
# Principal quantities (Section 4.1)
# ---------------------------------------------------------------------------------------------

@dataclass
class Quantities:
    alpha: list
    beta: list
    gamma: list
    a: list
    b: list
    q: list
    Q: Fraction
    e: list
    E: Fraction
    nnz: int


def quantities(rule: Rule) -> Quantities:
    R = rule.R
    nz = lambda x: 1 if x != 0 else 0
    alpha = [sum(nz(rule.U[i][r]) for i in range(len(rule.U))) for r in range(R)]  # eqn:abg
    beta = [sum(nz(rule.V[j][r]) for j in range(len(rule.V))) for r in range(R)]
    gamma = [sum(nz(rule.W[k][r]) for r in range(R)) for k in range(len(rule.W))]
    a = [sum(abs(rule.U[i][r]) for i in range(len(rule.U))) for r in range(R)]  # eqn:ab
    b = [sum(abs(rule.V[j][r]) for j in range(len(rule.V))) for r in range(R)]
    # Def. prefactor (eqn:qmax): q_k = gamma_k + max_r (alpha_r + beta_r) I(w_kr != 0)
    q = [gamma[k] + max((alpha[r] + beta[r]) * nz(rule.W[k][r]) for r in range(R))
         for k in range(len(rule.W))]
    # Def. stability (eqn:emax): e_k = sum_r a_r b_r |w_kr|
    e = [sum(a[r] * b[r] * abs(rule.W[k][r]) for r in range(R)) for k in range(len(rule.W))]
    nnz = sum(nz(x) for X in (rule.U, rule.V, rule.W) for row in X for x in row)
    return Quantities(alpha, beta, gamma, a, b, q, max(q), e, max(e), nnz)


def stationary_bound_factor(rule: Rule, L: int, K: int) -> Fraction:
    """Thm stationary_analysis: (K/K0^L + Q L)(K/K0^L) E^L."""
    qq = quantities(rule)
    kl = Fraction(K, rule.k0 ** L)
    return (kl + qq.Q * L) * kl * qq.E ** L


def uniform_bound_factor(rules: Sequence[Rule], K: int) -> Fraction:
    """Thm non_stationary_analysis: (K/prod K0 + sum Q)(K/prod K0) prod E."""
    pk = 1
    sq = Fraction(0)
    pe = Fraction(1)
    for r in rules:
        qq = quantities(r)
        pk *= r.k0
        sq += qq.Q
        pe *= qq.E
    kl = Fraction(K, pk)
    return (kl + sq) * kl * pe


def xi_nonuniform(plan_rules: list) -> Fraction:
    """Largest intermediate growth xi = max_k xi_k for a non-uniform plan (simplified
    form): plan_rules[l] is the list of rules of level l in BFS order (level 0 = root, one rule).
    xi_k = sum_{r1} |w^{[1]}_{k1 r1}| a_{r1} b_{r1} * sum_{r2} |w^{[2,r1]}_{k2 r2}| a b * ..."""
    L = len(plan_rules)

    def node_vec(level: int, idx: int) -> list:
        """Vector over the flattened k = (k_level, ..., k_L) of the subtree's growth."""
        rule = plan_rules[level][idx]
        qq = quantities(rule)
        out = []
        for kl in range(len(rule.W)):
            if level == L - 1:
                out.append([sum(abs(rule.W[kl][r]) * qq.a[r] * qq.b[r] for r in range(rule.R))])
            else:
                acc = None
                for r in range(rule.R):
                    c = abs(rule.W[kl][r]) * qq.a[r] * qq.b[r]
                    if c == 0:
                        continue
                    child = node_vec(level + 1, idx * rule.R + r)
                    flat = [c * x for x in child]
                    acc = flat if acc is None else [p + q for p, q in zip(acc, flat)]
                if acc is None:
                    acc = [Fraction(0)] * len(node_vec(level + 1, idx * rule.R))
                out.append(acc)
        return [x for sub in out for x in sub]

    return max(node_vec(0, 0))


def xi_nonuniform_full(plan_rules: list) -> Fraction:
    """xi = max_k xi_k by the unsimplified definition: for every root-to-leaf path
    (r_1, ..., r_L), |prod_l W^{[l]}_{k_l r_l}| * sum_{i_1..i_L} |prod_l U^{[l]}_{i_l r_l}|
    * sum_{j_1..j_L} |prod_l V^{[l]}_{j_l r_l}|, summed over paths; k = (k_1, ..., k_L)."""
    L = len(plan_rules)
    paths = [((), 0)]  # (r path, node index at the current level)
    nodes_on_path = {(): []}
    for level in range(L):
        nxt = []
        for path, idx in paths:
            rule = plan_rules[level][idx]
            for r in range(rule.R):
                np_ = path + (r,)
                nodes_on_path[np_] = nodes_on_path[path] + [rule]
                nxt.append((np_, idx * rule.R + r))
        paths = nxt
    kdims = [len(plan_rules[l][0].W) for l in range(L)]
    best = Fraction(0)
    for ks in product(*[range(d) for d in kdims]):
        total = Fraction(0)
        for path, _ in paths:
            rules_ = nodes_on_path[path]
            w = Fraction(1)
            for rule, k, r in zip(rules_, ks, path):
                w *= abs(rule.W[k][r])
            if w == 0:
                continue
            su = Fraction(0)
            for iis in product(*[range(len(rule.U)) for rule in rules_]):
                t = Fraction(1)
                for rule, i, r in zip(rules_, iis, path):
                    t *= abs(rule.U[i][r])
                su += t
            sv = Fraction(0)
            for jjs in product(*[range(len(rule.V)) for rule in rules_]):
                t = Fraction(1)
                for rule, j, r in zip(rules_, jjs, path):
                    t *= abs(rule.V[j][r])
                sv += t
            total += w * su * sv
        best = max(best, total)
    return best


def delta_nonuniform(plan_rules: list, K: int) -> Fraction:
    """Largest accumulation error delta = max_k delta_k^{[1]}, written out as the
    paper's recursion: delta_k^{[1]} = K/prod K0 + gamma_{k1} + max_{r1} delta_k^{[2,r1]}
    I(W_{k1 r1} != 0); inner levels gamma_{kl} + max_{rl} delta^{[l+1,..]}_k I(.); the last level
    gamma_{kL} + max_{rL} chi_r I(W_{kL rL} != 0), chi_r = sum over the path of alpha + beta."""
    L = len(plan_rules)
    pk = 1
    for lvl in plan_rules:
        pk *= lvl[0].k0
    kdims = [len(plan_rules[l][0].W) for l in range(L)]

    def delta(level, idx, ks, chi):
        rule = plan_rules[level][idx]
        qq = quantities(rule)
        k = ks[level]
        terms = []
        for r in range(rule.R):
            if rule.W[k][r] == 0:
                continue
            c = chi + qq.alpha[r] + qq.beta[r]
            terms.append(c if level == L - 1 else delta(level + 1, idx * rule.R + r, ks, c))
        return qq.gamma[k] + (max(terms) if terms else 0)

    return max(Fraction(K, pk) + delta(0, 0, ks, 0) for ks in product(*[range(d) for d in kdims]))


# ---------------------------------------------------------------------------------------------
# Plans
# ---------------------------------------------------------------------------------------------

@dataclass
class Plan:
    """levels[l] = list of rules for the nodes of level l in BFS order (len = prod R of levels
    above).  Stationary / uniform plans repeat one rule per level; non-uniform plans
     vary within a level but keep (M0,K0,N0,R)."""
    levels: list = field(default_factory=list)

    @property
    def L(self) -> int:
        return len(self.levels)

    @staticmethod
    def uniform(rules: Sequence[Rule]) -> "Plan":
        levels, n = [], 1
        for r in rules:
            levels.append([r] * n)
            n *= r.R
        return Plan(levels)

    @staticmethod
    def stationary(rule: Rule, L: int) -> "Plan":
        return Plan.uniform([rule] * L)

    @staticmethod
    def dalberto_two_level() -> "Plan":
        """The D'Alberto example: variant at nodes [2,1],[2,3],[2,4] (1-based r1),
        Strassen at [1],[2,2],[2,5],[2,6],[2,7]."""
        s, d = strassen(), strassen_dalberto()
        lvl2 = [d if r1 in (0, 2, 3) else s for r1 in range(7)]
        return Plan([[s], lvl2])

    def validate(self):
        n = 1
        for l, lv in enumerate(self.levels):
            assert len(lv) == n, f"level {l}: {len(lv)} rules, expected {n}"
            d = (lv[0].m0, lv[0].k0, lv[0].n0, lv[0].R)
            assert all((r.m0, r.k0, r.n0, r.R) == d for r in lv), "non-uniform dims within a level"
            n *= d[3]

    def dims_divisor(self):
        pm = pk = pn = 1
        for lv in self.levels:
            pm *= lv[0].m0
            pk *= lv[0].k0
            pn *= lv[0].n0
        return pm, pk, pn
