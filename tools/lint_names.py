"""Tiny undefined-name check (no linters in the image): flags names that are
read somewhere in a module but never bound anywhere in it."""
import ast
import builtins
import sys
from pathlib import Path


def check(path: Path) -> list[str]:
    tree = ast.parse(path.read_text())
    bound = set(dir(builtins)) | {"__file__", "__name__"}
    for node in ast.walk(tree):
        if isinstance(node, (ast.FunctionDef, ast.AsyncFunctionDef, ast.ClassDef)):
            bound.add(node.name)
        if isinstance(node, (ast.FunctionDef, ast.AsyncFunctionDef, ast.Lambda)):
            a = node.args
            for arg in a.args + a.kwonlyargs + a.posonlyargs + [a.vararg, a.kwarg]:
                if arg is not None:
                    bound.add(arg.arg)
        elif isinstance(node, (ast.Import, ast.ImportFrom)):
            for al in node.names:
                bound.add((al.asname or al.name).split(".")[0])
        elif isinstance(node, ast.Name) and isinstance(node.ctx, (ast.Store, ast.Del)):
            bound.add(node.id)
        elif isinstance(node, ast.ExceptHandler) and node.name:
            bound.add(node.name)
    out = []
    for node in ast.walk(tree):
        if isinstance(node, ast.Name) and isinstance(node.ctx, ast.Load) and node.id not in bound:
            out.append(f"{path}:{node.lineno}: undefined name {node.id!r}")
    return out


if __name__ == "__main__":
    errs = []
    for arg in sys.argv[1:]:
        p = Path(arg)
        for f in ([p] if p.is_file() else sorted(p.rglob("*.py"))):
            errs += check(f)
    print("\n".join(errs) or "ok")
    sys.exit(1 if errs else 0)
