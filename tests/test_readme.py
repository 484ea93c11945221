"""The README's quick-start snippet runs as written (GPU)."""
import os
import re

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def test_readme_quick_start():
    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "README.md")).read()
    code = re.search(r"```python\n(.*?)```", src, re.S).group(1)
    exec(compile(code, "README.md", "exec"), {})
