// Device-side encoding of a compiled rewrite program (the reference's
// DispatchTable, proj/include/trs/dispatch.hpp:73-78), packed into one blob
// that every CTA of the step loop copies into shared memory.
//
// Besides the reference fields, each rule carries the *subscription plan*
// of its RHS template: which freshly built node waits on which other fresh
// node.  A constructive rewrite at sweep s writes nodes that the reference
// would first inspect at sweep s+1, where every bound-variable child is
// already nf and every fresh child is not; so each fresh
// node's first fresh child (in argument order) is exactly the child its
// sweep-(s+1) subterm scan (sweep_engine.cpp:173-178) stops on.  The engine
// records that wait at build time instead of re-discovering it one sweep
// later.  Nodes with no fresh child go on the next sweep's frontier list.
#pragma once

#include <cstdint>

namespace trs_b200 {

constexpr uint32_t kSymBits = 24;
constexpr uint32_t kSymMask = (1u << kSymBits) - 1;
constexpr uint32_t kDeadHead = 0xFFFFFFFFu;  // head word of a collected slot
constexpr uint32_t kWoken = 0xFFFFFFFFu;     // waiter word: node is nf, do not sleep on it
constexpr uint8_t kNone = 0xFF;
constexpr uint8_t kRootSub = 0xFE;

constexpr uint32_t kMaxRuleSteps = 48;
constexpr uint32_t kMaxRuleInstrs = 32;
constexpr uint32_t kMaxVars = 48;  // binding columns live in dynamic shared memory (2 KB each)
constexpr uint32_t kMaxProgramBytes = 40 * 1024;

// record word layout (W words per slot, W = 8/16/32):
//   w0 head = symbol | subterm cursor << 24
//   w1 nf epoch: the sweep in which the slot became nf; while it is not nf,
//      kTminBit | the first sweep it may derive in (one past its build or
//      last in-place rewrite), or 0 for an input slot (the run's first sweep)
//   w2 refcount
//   w3 waiter (slot of the parent sleeping on this one, 0 none, kWoken)
//   w4.. arguments
constexpr uint32_t kWHead = 0, kWEpoch = 1, kWRc = 2, kWWaiter = 3, kWArgs = 4;
constexpr uint32_t kTminBit = 0x80000000u;
// An nf epoch word also carries the physical sweep that published it, mod 16
// (bits 27..30): with run-ahead (sweep.cuh) a lane may read records written
// in the current physical sweep only if it wrote them itself, so a child
// published in the current physical sweep by another lane counts as pending.
constexpr uint32_t kEpochBits = 27;
constexpr uint32_t kEpochMask = (1u << kEpochBits) - 1;
constexpr uint32_t kStampMask = 0xFu;

// Logical time (oracle/trs_oracle.c, oracle_logical): a slot derives in
// sweep T = max(its earliest sweep, max over arguments of their nf epoch + 1)
// (sweep_engine.cpp:80-81, :86, :153-188), whenever it is processed.
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr bool epoch_nf(uint32_t e) { return e != 0u && !(e & kTminBit); }

// Arguments a W-word record carries.  W = 16 holds at most 8 (not 12): the
// step loop keeps per-argument state in registers, and arity 9-12 systems
// are rare enough to take the 32-word layout instead.
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr int rec_args(int W) { return W == 16 ? 8 : W - 4; }

struct DRule {
    uint16_t first_step;
    uint8_t num_steps;
    uint8_t num_vars;
    uint16_t first_instr;
    uint8_t num_instrs;
    uint8_t new_slots;
    uint16_t root_ref;   // bit 15: node ref, else var slot
    uint8_t collapse;
    uint8_t root_wait;   // fresh instr the rewritten root sleeps on (kNone: push root)
    uint8_t root_cursor; // argument position of that wait
    uint8_t csrc;        // collapse source already in registers (kSrc* code of its binding step) or kNone
    uint8_t pad[2];
    uint32_t push_mask;  // bit k: fresh instr k goes on the next frontier list
};
static_assert(sizeof(DRule) == 20, "DRule layout");

struct DStep {
    uint8_t kind;  // 0 CheckHead, 1 BindVar
    uint8_t child;
    int8_t parent; // step index within the rule, -1 = redex root
    uint8_t src;   // where the level-synchronous matcher finds the value (kSrc*), see DPlan
    uint32_t value;
};
static_assert(sizeof(DStep) == 8, "DStep layout");

struct DInstr {
    uint32_t symbol;
    uint16_t first_ref;
    uint8_t indegree;
    uint8_t subscriber;  // who sleeps on this fresh node: kNone, kRootSub or instr index
    uint8_t cursor;      // argument position this node itself waits at
    uint8_t pad[3];
};
static_assert(sizeof(DInstr) == 12, "DInstr layout");

constexpr uint16_t kRefNode = 0x8000;

// Level-synchronous matching plan of one symbol.  The interpreted matcher
// walks each rule's steps in order (run_match_program, dispatch.hpp:95-117),
// one dependent gather per step below the root, and lanes of a warp trying
// different rules serialise those chains.  With a plan every lane instead
// issues the same loads at the same point: level 1 the redex's children
// (head, nf epoch and -- for the first kPlanChildren children, when listed
// in `child_args` -- their first four arguments, all in the child's first
// sector), level 2 the records of up to kPlanSlots grandchildren `slot_jk`
// (= child j's argument k), of which the first kPlanArgSlots may also bring
// their arguments.  (The limits keep the matcher's registers below the
// occupancy budget; they cover every pattern of the BASELINE systems.)  Every step of every rule of the
// symbol then reads its value from registers (DStep::src):
//   CheckHead  kSrcChild + c   head of child c
//              kSrcSlot + s    head of slot s
//   BindVar    kSrcChild + c   child c (the redex's argument)
//              kSrcCArg + 4j+k argument k of child j
//              kSrcSArg + 4s+k argument k of slot s
// Symbols whose rules reach deeper (or past these limits) keep the
// interpreted matcher (fast = 0).
constexpr uint8_t kSrcChild = 0x00, kSrcSlot = 0x40, kSrcCArg = 0x80, kSrcSArg = 0xC0;
constexpr uint8_t kPlanFast = 1, kPlanTables = 2;
constexpr uint16_t kNoRow = 0xFFFF;
// Match tables (planned symbols with <= 32 rules): rule choice without
// walking the rules.  Every CheckHead of a planned symbol reads a position
// -- child c's head (position c) or slot s's head (position rec_args(W)+s) --
// and row[p][h] is the mask of the symbol's rules that accept head h at
// position p (rules not checking p accept every h).  The first rule in
// source order whose checks all hold (dispatch.hpp:119-130) is the lowest
// bit of the AND over the checked positions.
constexpr uint32_t kPlanSlots = 2, kPlanArgSlots = 1, kPlanChildren = 2;

struct DPlan {
    uint8_t fast;        // bit 0: planned loads; bit 1: rule choice by match tables
    uint8_t child_args;  // bit j: load child j's first argument quad
    uint8_t nslots;
    uint8_t slot_args;   // bit s (s < kPlanArgSlots): load slot s's first argument quad
    uint8_t slot_jk[4];
};
static_assert(sizeof(DPlan) == 8, "DPlan layout");

// Constant chains.  A constant f() whose first rule (an arity-0 left-hand
// side always matches) rewrites it in place into another constant g(),
// building nothing, takes its next rewrites without looking at anything
// else: f -> g -> ... at consecutive logical sweeps.  chain[f] = g for such
// a step, kChainNf when f has no rules (it becomes nf), kChainNone otherwise.
// The run-ahead build takes a whole chain in registers (transform's leaves:
// A() -> B() -> ... -> End(), 26 rewrites, generators.cpp:84-110).
constexpr uint16_t kChainNone = 0xFFFF, kChainNf = 0xFFFE;
constexpr uint32_t kChainMax = 4096;

struct ProgHeader {
    uint32_t num_symbols;
    uint32_t num_rules;
    uint32_t num_steps;
    uint32_t num_instrs;
    uint32_t num_refs;
    uint32_t max_arity;
    uint32_t max_new_slots;
    uint32_t off_arity;       // uint8_t[num_symbols]
    uint32_t off_rule_begin;  // uint16_t[num_symbols + 1]
    uint32_t off_rules;       // DRule[]
    uint32_t off_steps;       // DStep[]
    uint32_t off_instrs;      // DInstr[]
    uint32_t off_refs;        // uint16_t[]
    uint32_t off_plans;       // DPlan[num_symbols]
    uint32_t off_mrow;        // uint16_t[num_symbols][npos]: match-table row per checked position, 0xFFFF none
    uint32_t off_mtab;        // uint32_t rows of num_symbols rule masks
    uint32_t npos;            // positions per symbol: rec_args(W) children + kPlanSlots slots (0: no tables)
    uint32_t off_chain;       // uint16_t[num_symbols]: constant chains (kChain*), see below
    uint32_t chains;          // the program has at least one constant-chain step
    uint32_t bytes;           // total blob size (multiple of 16)
};

}  // namespace trs_b200
