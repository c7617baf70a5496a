"""Second name shim (test infrastructure): the reference's `kvoverlap.numerics` mapped onto this repo's
CPU oracle (oracle/numerics_ref.py), so the reference's own numerics tests pin the oracle that every GPU
parity test is judged against (tests/test_reference_suite_cpu.py, R2).  The other modules map to the
package as in tests/refshim."""
