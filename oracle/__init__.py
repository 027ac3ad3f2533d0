"""TEST INFRASTRUCTURE ONLY: the CPU oracle (C restatement + reference build)."""
