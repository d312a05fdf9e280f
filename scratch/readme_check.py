import re, sys
sys.path.insert(0, '.')
src = open('README.md').read()
code = re.findall(r"```python\n(.*?)```", src, re.S)[-1]
exec(code)
