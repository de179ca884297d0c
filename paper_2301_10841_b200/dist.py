"""Multi-GPU sharding (north_star (c)): placeholder, implemented in the next step."""
