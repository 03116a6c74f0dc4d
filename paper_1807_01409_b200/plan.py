"""Query-plan types at the boundary: what ``evaluate_query`` consumes.

The SPARQL-subset parser itself is host string work and out of scope
(``sparql.py``); its OUTPUT types are the input of the hot path.
These dataclasses carry the same fields and helpers as reference
sparql.py:49-133 (Var, Term, TriplePattern, Filter, Group) and
sparql.py:372-425 (CompiledGroup, CompiledQuery, compile_group, compile_keys),
so objects produced by the reference parser work unchanged here (all access is
by attribute) and tests can build plans without it.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .kernel import PatternKey

SLOT_LETTERS = ("S", "P", "O")


@dataclass(frozen=True, slots=True)
class Var:
    name: str


@dataclass(frozen=True, slots=True)
class Term:
    lexical: str


def is_var(slot) -> bool:
    return hasattr(slot, "name")


@dataclass(frozen=True)
class TriplePattern:
    s: object
    p: object
    o: object

    @property
    def slots(self):
        return (self.s, self.p, self.o)

    @property
    def pattern_class(self) -> str:
        return "".join("?" if is_var(x) else SLOT_LETTERS[i] for i, x in enumerate(self.slots))

    def variables(self) -> list[str]:
        names: list[str] = []
        for x in self.slots:
            if is_var(x) and x.name not in names:
                names.append(x.name)
        return names

    def var_slots(self) -> dict[str, list[int]]:
        where: dict[str, list[int]] = {}
        for i, x in enumerate(self.slots):
            if is_var(x):
                where.setdefault(x.name, []).append(i)
        return where


@dataclass(frozen=True)
class Filter:
    variable: str
    regex: str


@dataclass
class Group:
    patterns: list
    filters: list

    def variables(self) -> list[str]:
        names: list[str] = []
        for pat in self.patterns:
            for v in pat.variables():
                if v not in names:
                    names.append(v)
        return names


@dataclass
class CompiledGroup:
    patterns: list
    filters: list
    keys: list
    var_slots: list
    satisfiable: bool
    variables: list = field(default_factory=list)


@dataclass
class CompiledQuery:
    groups: list
    distinct: bool
    projection: list | None
    output_columns: list


def compile_group(group, dictionary) -> CompiledGroup:
    """Terms -> IDs, variables -> 0; an unknown term makes the group
    unsatisfiable (sparql.py:396-419)."""
    keys = []
    ok = True
    for pat in group.patterns:
        ids = []
        for x in pat.slots:
            if is_var(x):
                ids.append(0)
                continue
            ident = dictionary.lookup(x.lexical)
            if ident is None:
                ok = False
                ident = 0
            ids.append(ident)
        keys.append(PatternKey(*ids))
    return CompiledGroup(
        patterns=list(group.patterns),
        filters=list(group.filters),
        keys=keys,
        var_slots=[pat.var_slots() for pat in group.patterns],
        satisfiable=ok,
        variables=group.variables(),
    )


def compile_query(groups, dictionary, *, distinct: bool = False,
                  projection: list | None = None) -> CompiledQuery:
    """Lower a list of Groups (the parser's QueryAst.groups) against a dictionary."""
    compiled = [compile_group(g, dictionary) for g in groups]
    cols: list[str] = []
    for g in groups:
        for v in g.variables():
            if v not in cols:
                cols.append(v)
    return CompiledQuery(compiled, distinct, projection,
                         list(projection) if projection is not None else cols)


def compile_keys(ast, dictionary) -> CompiledQuery:
    """Same as reference sparql.compile_keys for a parsed QueryAst."""
    return compile_query(ast.groups, dictionary, distinct=ast.distinct,
                         projection=ast.projection)


# -- small helpers for building plans in code ----------------------------------

def V(name: str) -> Var:
    return Var(name)


def T(lexical: str) -> Term:
    return Term(lexical)


def pattern(s, p, o) -> TriplePattern:
    """Slots given as '?x' strings (variables) or lexical term strings."""
    conv = [Var(x[1:]) if isinstance(x, str) and x.startswith("?") else
            (Term(x) if isinstance(x, str) else x) for x in (s, p, o)]
    return TriplePattern(*conv)
