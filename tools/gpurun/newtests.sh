timeout 900 python -m pytest tests -m gpu -x -q -k "holes or disconnected or wheels" 2>&1 | tail -5
