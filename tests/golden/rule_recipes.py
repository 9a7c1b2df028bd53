"""Custom classify rule tables from JSON recipes, shared by the fixture
generator (reference predicates) and the GPU test (device predicates).

A recipe entry is [op, *args, label]:
  ["b", mode_id, label]       the builtin predicate of mode_id, relabelled
  ["size_ge", n, label]       c.size >= n
  ["has", kind, label]        c.has(kind)
  ["last_lt", a, b, label]    c.last(a) < c.last(b)
  ["d0_none", label]          c.d0 is None
  ["true", label] / ["false", label]
"""


def _host_pred(op, args, event_kind):
    if op == "size_ge":
        return lambda c, n=args[0]: c.size >= n
    if op == "has":
        return lambda c, k=event_kind(args[0]): c.has(k)
    if op == "last_lt":
        return lambda c, a=event_kind(args[0]), b=event_kind(args[1]): c.last(a) < c.last(b)
    if op == "d0_none":
        return lambda c: c.d0 is None
    if op == "true":
        return lambda c: True
    if op == "false":
        return lambda c: False
    raise ValueError(op)


def build_table(recipe, builtin_rules, subtask_kind, event_kind):
    """recipe = {subtask_value: {"success": [...], "failure": [...]}} -> a
    classify rules table; builtin_rules = that implementation's MODE_RULES."""
    table = {}
    for sub, branches in recipe.items():
        k = subtask_kind(sub)
        own = {m: p for br in ("success", "failure") for m, p in builtin_rules[k][br]}
        out = {}
        for br in ("success", "failure"):
            rows = []
            for ent in branches[br]:
                op, args, label = ent[0], ent[1:-1], ent[-1]
                pred = own[args[0]] if op == "b" else _host_pred(op, args, event_kind)
                rows.append((label, pred))
            out[br] = rows
        table[k] = out
    return table
