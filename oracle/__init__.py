"""Test-infrastructure oracle (CPU restatement of the reference path). See star_oracle.py."""
