"""REXII hot path on B200 (sm_100a). The CUDA library is loaded lazily by paper_2008_11607_b200.rexi."""
