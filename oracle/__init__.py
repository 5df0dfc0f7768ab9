# ORACLE — TEST INFRASTRUCTURE ONLY (CPU restatement of the reference; see h2oracle.hpp).
