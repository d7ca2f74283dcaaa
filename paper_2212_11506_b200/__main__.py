"""`python -m paper_2212_11506_b200 embed|profile|kl ...` (the CLI in cli.py)."""

from paper_2212_11506_b200 import cli

raise SystemExit(cli.main())
