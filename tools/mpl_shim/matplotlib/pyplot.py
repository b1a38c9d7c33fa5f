"""No-op pyplot for the reference CLI tests (see __init__.py)."""


class _Any:
    def __getattr__(self, name):
        return lambda *a, **k: None


class _Fig(_Any):
    def savefig(self, path, *a, **k):
        with open(path, "wb") as fh:
            fh.write(b"\x89PNG placeholder")


def subplots(nrows=1, ncols=1, **k):
    axes = _Any() if nrows * ncols == 1 else tuple(_Any() for _ in range(nrows * ncols))
    return _Fig(), axes


def close(*a, **k):
    return None
