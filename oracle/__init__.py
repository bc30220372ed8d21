"""CPU oracle for the foveation hot path -- test infrastructure only (see fovea_oracle.py)."""
