"""Runs the reference's OWN test-suite (baseline/_ref/tests, unmodified) against the
drop-in: test infrastructure only (see alias_plugin.py)."""
