"""Host offline stage (restated reference, layer-parallel) and BASELINE configs."""
