"""Mutation check of the oracle pins (`-m "not gpu"`): every plausible mistake
listed in scripts/oracle_mutants.py (delay off by one, reversed slice mapping,
flipped spatial index, dropped history push, the printed Principle-6
recurrence, head / stride-phase / ring-size / grouping / padding / bias / bf16
rounding errors) must fail at least one pin in tests/test_oracle_pins.py."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def test_every_oracle_mutant_is_killed(capsys):
    if os.environ.get("CO_ORACLE_LIB"):      # running inside the mutation check itself
        return
    import oracle_mutants
    rc = oracle_mutants.main([])
    out = capsys.readouterr().out
    assert rc == 0, out
    assert out.count("killed ") == len(oracle_mutants.MUTANTS), out
