"""CPU oracle for one coarsening level — TEST INFRASTRUCTURE ONLY (see hgp_ref.h)."""
