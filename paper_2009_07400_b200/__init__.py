"""tinyMD pairwise-interaction timestep on B200 (placeholder during bring-up)."""
