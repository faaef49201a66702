"""Oracle package -- TEST INFRASTRUCTURE ONLY (see asyflexa_oracle.py header)."""
