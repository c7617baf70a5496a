"""Name shim (test infrastructure): the reference's package name over this package's modules, so the
reference's own test files (/root/reference/pkg/tests) run unmodified against the drop-in
(tests/test_reference_suite_cpu.py).  Nothing here is imported by the product."""
