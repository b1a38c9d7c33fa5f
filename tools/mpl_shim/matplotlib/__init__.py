"""Test-only stand-in for matplotlib (not installed in this image), so the
reference's CLI tests can run: every drawing call is a no-op and savefig
writes a placeholder file.  Used only by tools/ref_suite_plugin runs."""


def use(backend):
    return None
