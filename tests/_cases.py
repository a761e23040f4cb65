"""Shared helpers: load golden fixtures and rebuild the bundle of a case."""
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def build(mod, case):
    fn, args, kw = case
    args = [tuple(a) if isinstance(a, list) else a for a in args]
    kw = {k: tuple(v) if isinstance(v, list) else v for k, v in kw.items()}
    return getattr(mod, fn)(*args, **kw)


def case_id(case):
    fn, args, kw = case
    return f"{fn}{args}{kw.get('dims', '')}{'c' + str(kw['chunk']) if 'chunk' in kw else ''}".replace(" ", "")
