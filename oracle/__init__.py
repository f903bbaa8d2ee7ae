"""CPU ORACLE — test infrastructure only.

Imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg, and there only as the checker or the
CPU baseline. The product package (paper_2302_02599_b200) never imports it.

  oracle.ref   ctypes over oracle/_ref/libautoplan_ref.so, the REFERENCE
               autoplan library compiled from /root/reference sources
               (oracle/Makefile); spec-level truth (paths, costs, specs).
  oracle.data  ctypes over oracle/_build/libapl_oracle.so, the plain-C
               restatement of the step data semantics (apl_oracle.c).
"""
from pathlib import Path

HERE = Path(__file__).resolve().parent


def build(ref: bool = True) -> None:
    """Build the C restatement and, when /root/reference exists, the
    reference library (building the checker is not using it)."""
    import subprocess

    # "in_memory": the reference planner TUs linked against the built
    # libapl.so (tests/cpp/plan_in_memory_test.cpp), so build() runs it last
    targets = ["all", "in_memory"] if ref and Path("/root/reference/proj/src").exists() else [
        str(HERE / "_build" / "libapl_oracle.so")]
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)
